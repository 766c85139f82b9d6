// A C++ caller that reads the reference's whole RoutingPlan surface (routing.hpp:93-170):
// routes[*].params / .optim CategorySets (src, dst, send, recv, retain), route_of(),
// the unresolved `pending` fragments with their candidates, the ScalarBroadcast, then the
// resolved transfers, bytes_moved() and bytes_retained(space).
//
// The same file compiles against the reference headers (-DREF_D1_SHIM, the golden
// generator in tests/golden/make_golden.py via oracle/Makefile) and against this repo's
// (tests/test_cpp_routing.py); their outputs must be identical.
//
//   routes_dump <scenario file>   (exit 2 + "# error: ..." on ConfigError)
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>

#include "reshard/common.hpp"
#include "reshard/model.hpp"
#include "reshard/parallel.hpp"
#include "reshard/project.hpp"
#include "reshard/region.hpp"
#include "reshard/topology.hpp"
#include "reshard/worldmap.hpp"

#ifdef REF_D1_SHIM
// routing.hpp:389 dereferences a null ModelSpace (D1): while the reference header is
// parsed, `nullptr` names the address of the live space instead (oracle/ref_plan.cpp)
inline std::uintptr_t reshard_d1_space_addr = 0;
#define nullptr reshard_d1_space_addr
#include "reshard/routing.hpp"
#undef nullptr
#else
#include "reshard/routing.hpp"
#endif

#include "scenario_text.hpp"

using namespace reshard;

static std::string out;

static void line(const std::string& s) {
    out += s;
    out += '\n';
}

static void region(const char* what, const RegionSet& r) {
    for (const auto& [id, boxes] : r.boxes)
        for (const Box& b : boxes) line(strfmt("  %s box %s %s", what, id.c_str(), format_box(b).c_str()));
    for (const Interval& i : r.flat) line(strfmt("  %s flat %s", what, format_interval(i).c_str()));
}

static void category(const char* name, const CategorySet& c) {
    const std::string n(name);
    region((n + ".src").c_str(), c.src);
    region((n + ".dst").c_str(), c.dst);
    region((n + ".send").c_str(), c.send);
    region((n + ".recv").c_str(), c.recv);
    region((n + ".retain").c_str(), c.retain);
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: routes_dump <scenario>\n");
        return 2;
    }
    try {
        std::ifstream f(argv[1]);
        if (!f) throw ConfigError(std::string("cannot open ") + argv[1]);
        const reshard_text::Scenario sc = reshard_text::parse_scenario(f);
        const ModelSpace space = build_model_space(sc.model);
        validate_config(sc.src, sc.model);
        validate_config(sc.dst, sc.model);
        const WorldMap wm = sc.wm ? *sc.wm : WorldMap::identity(sc.src.world_size(), sc.dst.world_size());
        RoutingPlan plan = plan_parameters(space, sc.src, sc.dst, wm, sc.opts);
        plan_optimizer(space, plan);
        plan_scalars(plan);
        for (const RankRoute& r : plan.routes) {
            line(strfmt("route phys=%d src=%d dst=%d", r.phys, r.src_rank, r.dst_rank));
            category("params", r.params);
            category("optim", r.optim);
            const RankRoute& again = plan.route_of(r.phys);
            line(strfmt("  route_of retain_flat=%lld", static_cast<long long>(again.optim.retain.flat_numel())));
        }
        for (const auto& p : plan.pending) {
            std::string c;
            for (int x : p.candidates) c += (c.empty() ? "" : ",") + std::to_string(x);
            line(strfmt("pending %s %s %s dst_phys=%d dst_rank=%d cands=%s", to_string(p.kind),
                        p.tensor_id.empty() ? "-" : p.tensor_id.c_str(),
                        p.flat_payload ? format_interval(p.flat).c_str() : format_box(p.box).c_str(), p.dst_phys,
                        p.dst_rank, c.c_str()));
        }
        if (plan.scalars) {
            std::string rp;
            for (int x : plan.scalars->recv_phys) rp += (rp.empty() ? "" : ",") + std::to_string(x);
            line(strfmt("scalars root_phys=%d root_src_rank=%d words=%lld bytes_per_rank=%lld recv=%s",
                        plan.scalars->root_phys, plan.scalars->root_src_rank, static_cast<long long>(plan.scalars->words),
                        static_cast<long long>(plan.scalars->bytes_per_rank), rp.c_str()));
        } else {
            line("scalars none");
        }
#ifdef REF_D1_SHIM
        reshard_d1_space_addr = reinterpret_cast<std::uintptr_t>(&space);
#endif
        resolve_peers(plan, sc.topo);
        line(strfmt("resolved=%d pending=%zu transfers=%zu bytes_moved=%lld bytes_retained=%lld", plan.resolved ? 1 : 0,
                    plan.pending.size(), plan.transfers.size(), static_cast<long long>(plan.bytes_moved()),
                    static_cast<long long>(plan.bytes_retained(space))));
        for (const SliceTransfer& t : plan.transfers)
            line(format_transfer(t) + strfmt(" src_phys=%d dst_phys=%d count=%lld", t.src_phys, t.dst_phys,
                                             static_cast<long long>(t.count)));
    } catch (const ConfigError& e) {
        std::fwrite(out.data(), 1, out.size(), stdout);
        std::printf("# error: %s\n", e.what());
        return 2;
    }
    std::fwrite(out.data(), 1, out.size(), stdout);
    return 0;
}
