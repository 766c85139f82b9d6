// ref_plan.cpp — drives the UNMODIFIED reference headers (/root/reference/proj/include)
// on a scenario file and prints the reference plan dump. Test infrastructure only:
// built by oracle/Makefile into oracle/_ref/ref_plan and used to pin the oracle
// restatement and to generate tests/golden/.
//
// D1 shim: routing.hpp:389 reinterpret_casts nullptr to a ModelSpace
// reference, which g++ rejects. We define `nullptr` as an integer holding the address
// of the live ModelSpace while (and only while) routing.hpp is parsed, so the call
// resolves the real dtype widths (routing.hpp:174-183). No reference line is edited.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "reshard/common.hpp"
#include "reshard/model.hpp"
#include "reshard/parallel.hpp"
#include "reshard/project.hpp"
#include "reshard/region.hpp"
#include "reshard/topology.hpp"
#include "reshard/worldmap.hpp"

inline std::uintptr_t reshard_d1_space_addr = 0;
#define nullptr reshard_d1_space_addr
#include "reshard/routing.hpp"
#undef nullptr

using namespace reshard;

struct Scenario {
    ModelSpec model;
    ParallelConfig src, dst;
    std::optional<WorldMap> wm;
    Topology topo;
    PlanOptions opts;
};

static std::vector<std::int64_t> parse_list(const std::string& s) {
    std::vector<std::int64_t> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) {
        if (item.empty()) throw ConfigError("bad list '" + s + "'");
        out.push_back(std::stoll(item));
    }
    return out;
}

static Scenario parse(std::istream& in) {
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

static int cmd_plan(const Scenario& sc) {
    ModelSpace space = build_model_space(sc.model);
    validate_config(sc.src, sc.model);
    validate_config(sc.dst, sc.model);
    WorldMap wm = sc.wm ? *sc.wm : WorldMap::identity(sc.src.world_size(), sc.dst.world_size());
    RoutingPlan plan = plan_parameters(space, sc.src, sc.dst, wm, sc.opts);
    plan_optimizer(space, plan);
    plan_scalars(plan);
    reshard_d1_space_addr = reinterpret_cast<std::uintptr_t>(&space);
    resolve_peers(plan, sc.topo);
    reshard_d1_space_addr = 0;
    std::string out;
    for (const auto& t : plan.transfers) {
        out += format_transfer(t);
        out += '\n';
    }
    std::fwrite(out.data(), 1, out.size(), stdout);
    std::printf("# transfers=%zu bytes_moved=%lld bytes_retained=%lld\n", plan.transfers.size(),
                static_cast<long long>(plan.bytes_moved()), static_cast<long long>(plan.bytes_retained(space)));
    return 0;
}

static int cmd_regions(const Scenario& sc, bool dst) {
    ModelSpace space = build_model_space(sc.model);
    const ParallelConfig& cfg = dst ? sc.dst : sc.src;
    validate_config(cfg, sc.model);
    for (int r = 0; r < cfg.world_size(); ++r) {
        RegionSet reg = project(space, cfg, r);
        for (const auto& [id, boxes] : reg.boxes)
            for (const auto& b : boxes) std::printf("rank %d param %s %s\n", r, id.c_str(), format_box(b).c_str());
        LocalLayout L = local_layout(space, cfg, r);
        for (const auto& s : L.dense)
            std::printf("rank %d layout dense %s %s %lld %lld\n", r, s.tensor_id.c_str(), format_box(s.box).c_str(),
                        static_cast<long long>(s.local_lo), static_cast<long long>(s.local_hi));
        for (const auto& s : L.expert)
            std::printf("rank %d layout expert %s %s %lld %lld\n", r, s.tensor_id.c_str(), format_box(s.box).c_str(),
                        static_cast<long long>(s.local_lo), static_cast<long long>(s.local_hi));
        if (cfg.zero_enabled) {
            RegionSet o = project_optimizer(space, cfg, r);
            for (const auto& iv : o.flat) std::printf("rank %d optim %s\n", r, format_interval(iv).c_str());
        }
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ref_plan plan|regions-src|regions-dst <scenario|->\n");
        return 2;
    }
    try {
        Scenario sc;
        if (std::string(argv[2]) == "-") sc = parse(std::cin);
        else {
            std::ifstream f(argv[2]);
            if (!f) throw ConfigError(std::string("cannot open ") + argv[2]);
            sc = parse(f);
        }
        std::string cmd = argv[1];
        if (cmd == "plan") return cmd_plan(sc);
        if (cmd == "regions-src") return cmd_regions(sc, false);
        if (cmd == "regions-dst") return cmd_regions(sc, true);
        std::fprintf(stderr, "unknown command\n");
        return 2;
    } catch (const ConfigError& e) {
        std::fflush(stdout);
        std::printf("# error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fflush(stdout);
        std::printf("# internal: %s\n", e.what());
        return 1;
    }
}
