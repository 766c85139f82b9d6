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

#include "scenario_text.hpp"
using reshard_text::Scenario;

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
        if (std::string(argv[2]) == "-") sc = reshard_text::parse_scenario(std::cin);
        else {
            std::ifstream f(argv[2]);
            if (!f) throw ConfigError(std::string("cannot open ") + argv[2]);
            sc = reshard_text::parse_scenario(f);
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
