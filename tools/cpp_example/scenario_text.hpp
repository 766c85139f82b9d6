// Scenario text -> the reference API's value types. Uses only the
// reference's public types, so it compiles against the reference headers
// (oracle/ref_plan.cpp, the golden generator) and against this repo's (the C++ examples).
#pragma once

#include <cstdint>
#include <istream>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

namespace reshard_text {

using namespace reshard;

struct Scenario {
    ModelSpec model;
    ParallelConfig src, dst;
    std::optional<WorldMap> wm;
    Topology topo;
    PlanOptions opts;
};

inline std::vector<std::int64_t> parse_list(const std::string& s) {
    std::vector<std::int64_t> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) {
        if (item.empty()) throw ConfigError("bad list '" + s + "'");
        out.push_back(std::stoll(item));
    }
    return out;
}

inline Scenario parse_scenario(std::istream& in) {
    Scenario sc;
    std::string line;
    while (std::getline(in, line)) {
        std::stringstream ls(line);
        std::vector<std::string> tok;
        std::string w;
        while (ls >> w) tok.push_back(w);
        if (tok.empty() || tok[0][0] == '#' || tok[0] == "version" || tok[0] == "seed") continue;
        auto kv = [](const std::string& t) {
            auto eq = t.find('=');
            if (eq == std::string::npos) throw ConfigError("bad token '" + t + "'");
            return std::make_pair(t.substr(0, eq), t.substr(eq + 1));
        };
        if (tok[0] == "model") {
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "layers") sc.model.num_layers = std::stoi(v);
                else if (k == "experts") sc.model.num_experts = std::stoi(v);
                else throw ConfigError("bad model key");
            }
        } else if (tok[0] == "tensor") {
            TensorSpec t;
            t.tensor_id = tok.at(1);
            t.shape = parse_list(tok.at(2));
            for (size_t i = 3; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "layer") t.layer = std::stoi(v);
                else if (k == "tp") t.tp_shard_axis = std::stoi(v);
                else if (k == "expert") { t.expert_axis = std::stoi(v); t.is_expert = true; }
                else if (k == "dtype") t.dtype_bytes = std::stoi(v);
                else throw ConfigError("bad tensor key");
            }
            sc.model.tensors.push_back(t);
        } else if (tok[0] == "src" || tok[0] == "dst") {
            ParallelConfig& c = tok[0] == "src" ? sc.src : sc.dst;
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "dp") c.dp = std::stoi(v);
                else if (k == "tp") c.tp = std::stoi(v);
                else if (k == "pp") c.pp = std::stoi(v);
                else if (k == "ep") c.ep = std::stoi(v);
                else if (k == "zero") c.zero_enabled = std::stoi(v) != 0;
                else if (k == "order") c.rank_order = v;
                else throw ConfigError("bad config key");
            }
        } else if (tok[0] == "world") {
            WorldMap m;
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                auto l = v.empty() ? std::vector<std::int64_t>{} : parse_list(v);
                std::vector<int> li(l.begin(), l.end());
                if (k == "src") m.src_phys = li;
                else if (k == "dst") m.dst_phys = li;
                else throw ConfigError("bad world key");
            }
            sc.wm = m;
        } else if (tok[0] == "topology") {
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "nodes") sc.topo.num_nodes = std::stoi(v);
                else if (k == "rpn") sc.topo.ranks_per_node = std::stoi(v);
                else throw ConfigError("bad topology key");
            }
        } else if (tok[0] == "options") {
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "grads") sc.opts.gradients = v == "migrate" ? GradientPolicy::Migrate : GradientPolicy::Drop;
                else if (k == "balance") sc.opts.balance_fanout = std::stoi(v) != 0;
                else if (k == "scalar_words") sc.opts.scalar_words = std::stoll(v);
                else throw ConfigError("bad option");
            }
        } else {
            throw ConfigError("unknown keyword '" + tok[0] + "'");
        }
    }
    return sc;
}


}  // namespace reshard_text
