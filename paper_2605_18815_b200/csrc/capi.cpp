// C ABI (include/reshard_b200.h): thin, exception-free wrappers over the C++
// planner (reshard::core) and the executor (reshard::exec).
#include "reshard_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "reshard/arena.hpp"
#include "reshard/edm.hpp"
#include "reshard/fdx.hpp"
#include "reshard/nccl_comm.hpp"
#include "reshard/executor_rt.hpp"
#include "reshard/plan_core.hpp"
#include "reshard/schedule.hpp"
#include "reshard/sync.hpp"
#include "reshard/validate.hpp"

namespace reshard {
namespace gpuplan {
std::vector<core::FlatXfer> expand_flat_gpu(const core::PlanCore& P, int device, double* kernel_ms);
std::vector<core::BoxXfer> box_routes_gpu(const core::PlanCore& P, int device, double* kernel_ms);
}
}  // namespace reshard

using namespace reshard;

struct rs_model {
    ModelSpec spec;
    ModelSpace space;
};

struct rs_plan {
    std::shared_ptr<rs_model> owned;  // set when created from scenario text
    const rs_model* model = nullptr;
    core::PlanCore core;
};

struct rs_schedule {
    const rs_plan* plan = nullptr;
    sched::TransitionSchedule T;
};

struct rs_arena {
    std::unique_ptr<mem::Arena> a;
};

struct rs_sync {
    std::unique_ptr<sync::DeviceBarrier> b;
};

struct rs_exec {
    const rs_plan* plan = nullptr;
    std::unique_ptr<exec::Executor> ex;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const ConfigError& e) {
        return fail(RS_ERR_CONFIG, e.what());
    } catch (const exec::CudaError& e) {
        return fail(RS_ERR_CUDA, e.what());
    } catch (const exec::BudgetError& e) {
        return fail(RS_ERR_BUDGET, e.what());
    } catch (const std::bad_alloc&) {
        return fail(RS_ERR_INTERNAL, "out of host memory");
    } catch (const std::exception& e) {
        return fail(RS_ERR_INTERNAL, e.what());
    }
}

char* dup_string(const std::string& s, size_t* len) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (!p) throw std::bad_alloc();
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = 0;
    if (len) *len = s.size();
    return p;
}

ParallelConfig to_cfg(const rs_cfg_t& c) {
    ParallelConfig p;
    p.dp = c.dp;
    p.tp = c.tp;
    p.pp = c.pp;
    p.ep = c.ep;
    p.zero_enabled = c.zero != 0;
    if (c.order) p.rank_order = c.order;
    return p;
}

std::vector<std::int64_t> parse_ints(const std::string& s) {
    std::vector<std::int64_t> v;
    std::stringstream ss(s);
    std::string x;
    while (std::getline(ss, x, ','))
        if (!x.empty()) v.push_back(std::stoll(x));
    return v;
}

struct Scenario {
    ModelSpec model;
    ParallelConfig src, dst;
    bool has_world = false;
    WorldMap wm;
    Topology topo;
    PlanOptions opts;
};

/// Scenario text: the reference's value structs, one per line.
Scenario parse_scenario(const std::string& text) {
    Scenario sc;
    std::stringstream in(text);
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        std::stringstream ls(line);
        std::vector<std::string> tok;
        for (std::string w; ls >> w;) tok.push_back(w);
        if (tok.empty() || tok[0][0] == '#' || tok[0] == "version" || tok[0] == "seed") continue;
        auto kv = [&](const std::string& t) {
            const size_t eq = t.find('=');
            if (eq == std::string::npos) throw ConfigError(strfmt("line %d: bad token '%s'", lineno, t.c_str()));
            return std::make_pair(t.substr(0, eq), t.substr(eq + 1));
        };
        if (tok[0] == "model") {
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "layers") sc.model.num_layers = std::stoi(v);
                else if (k == "experts") sc.model.num_experts = std::stoi(v);
                else throw ConfigError(strfmt("line %d: bad model key", lineno));
            }
        } else if (tok[0] == "tensor") {
            if (tok.size() < 3) throw ConfigError(strfmt("line %d: tensor needs id and shape", lineno));
            TensorSpec t;
            t.tensor_id = tok[1];
            t.shape = parse_ints(tok[2]);
            for (size_t i = 3; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "layer") t.layer = std::stoi(v);
                else if (k == "tp") t.tp_shard_axis = std::stoi(v);
                else if (k == "expert") t.expert_axis = std::stoi(v), t.is_expert = true;
                else if (k == "dtype") t.dtype_bytes = std::stoi(v);
                else throw ConfigError(strfmt("line %d: bad tensor key", lineno));
            }
            sc.model.tensors.push_back(std::move(t));
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
                else throw ConfigError(strfmt("line %d: bad config key", lineno));
            }
        } else if (tok[0] == "world") {
            sc.has_world = true;
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                std::vector<std::int64_t> l = parse_ints(v);
                std::vector<int> li(l.begin(), l.end());
                if (k == "src") sc.wm.src_phys = li;
                else if (k == "dst") sc.wm.dst_phys = li;
                else throw ConfigError(strfmt("line %d: bad world key", lineno));
            }
        } else if (tok[0] == "topology") {
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "nodes") sc.topo.num_nodes = std::stoi(v);
                else if (k == "rpn") sc.topo.ranks_per_node = std::stoi(v);
                else throw ConfigError(strfmt("line %d: bad topology key", lineno));
            }
        } else if (tok[0] == "options") {
            for (size_t i = 1; i < tok.size(); ++i) {
                auto [k, v] = kv(tok[i]);
                if (k == "grads") sc.opts.gradients = v == "migrate" ? GradientPolicy::Migrate : GradientPolicy::Drop;
                else if (k == "balance") sc.opts.balance_fanout = std::stoi(v) != 0;
                else if (k == "scalar_words") sc.opts.scalar_words = std::stoll(v);
                else throw ConfigError(strfmt("line %d: bad option", lineno));
            }
        } else {
            throw ConfigError(strfmt("line %d: unknown keyword '%s'", lineno, tok[0].c_str()));
        }
    }
    return sc;
}

std::vector<core::FlatXfer> expand(const rs_plan* p, int device) {
    if (device >= 0) return gpuplan::expand_flat_gpu(p->core, device, nullptr);
    return core::expand_flat_host(p->core);
}

}  // namespace

extern "C" {

const char* rs_last_error(void) { return g_err.c_str(); }
const char* rs_version(void) { return "reshard-b200 0.1 (sm_100a)"; }
void rs_free(void* p) { std::free(p); }

int rs_model_create(const rs_tensor_t* tensors, int n, int num_layers, int num_experts, rs_model_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto m = std::make_unique<rs_model>();
        m->spec.num_layers = num_layers;
        m->spec.num_experts = num_experts;
        for (int i = 0; i < n; ++i) {
            const rs_tensor_t& t = tensors[i];
            if (!t.id || t.ndim < 1 || t.ndim > 4) throw ConfigError("tensor needs an id and 1..4 dims");
            TensorSpec s;
            s.tensor_id = t.id;
            s.shape.assign(t.shape, t.shape + t.ndim);
            s.layer = t.layer;
            if (t.tp_axis >= 0) s.tp_shard_axis = t.tp_axis;
            if (t.expert_axis >= 0) s.expert_axis = t.expert_axis, s.is_expert = true;
            s.dtype_bytes = t.dtype_bytes;
            m->spec.tensors.push_back(std::move(s));
        }
        m->space = build_model_space(m->spec);
        *out = m.release();
        return RS_OK;
    });
}

void rs_model_destroy(rs_model_t* m) { delete m; }

int rs_plan_create(const rs_model_t* m, const rs_cfg_t* src, const rs_cfg_t* dst, const rs_worldmap_t* wm,
                   const rs_topo_t* topo, const rs_options_t* opts, rs_plan_t** out) {
    return guarded([&] {
        *out = nullptr;
        if (!m || !src || !dst) throw ConfigError("null model or config");
        auto p = std::make_unique<rs_plan>();
        p->model = m;
        WorldMap w;
        if (wm) {
            w.src_phys.assign(wm->src_phys, wm->src_phys + wm->n_src);
            w.dst_phys.assign(wm->dst_phys, wm->dst_phys + wm->n_dst);
        }
        Topology t;
        if (topo) t.num_nodes = topo->num_nodes, t.ranks_per_node = topo->ranks_per_node;
        PlanOptions o;
        bool allow = false;
        if (opts) {
            o.gradients = opts->migrate_grads ? GradientPolicy::Migrate : GradientPolicy::Drop;
            o.balance_fanout = opts->balance_fanout != 0;
            o.scalar_words = opts->scalar_words;
            allow = opts->allow_oversourced != 0;
        }
        p->core = core::build_plan(m->space, to_cfg(*src), to_cfg(*dst), wm ? &w : nullptr, t, o, allow);
        *out = p.release();
        return RS_OK;
    });
}

int rs_plan_from_scenario(const char* text, int allow_oversourced, rs_plan_t** out) {
    return guarded([&] {
        *out = nullptr;
        Scenario sc = parse_scenario(text ? text : "");
        auto m = std::make_shared<rs_model>();
        m->spec = sc.model;
        m->space = build_model_space(m->spec);
        auto p = std::make_unique<rs_plan>();
        p->owned = m;
        p->model = m.get();
        p->core = core::build_plan(m->space, sc.src, sc.dst, sc.has_world ? &sc.wm : nullptr, sc.topo, sc.opts,
                                   allow_oversourced != 0);
        *out = p.release();
        return RS_OK;
    });
}

void rs_plan_destroy(rs_plan_t* p) { delete p; }

int rs_plan_summary(const rs_plan_t* p, rs_plan_summary_t* out) {
    return guarded([&] {
        std::memset(out, 0, sizeof *out);
        const core::PlanCore& c = p->core;
        out->num_box_transfers = static_cast<std::int64_t>(c.box.size());
        out->num_flat_transfers = c.n_flat;
        out->num_transfers = c.num_transfers();
        out->bytes_moved = c.bytes_moved;
        out->bytes_retained = c.bytes_retained;
        out->num_triples = static_cast<std::int64_t>(c.triples.size());
        out->src_world = c.src_cfg.world_size();
        out->dst_world = c.dst_cfg.world_size();
        out->num_participants = static_cast<int>(c.routes.size());
        out->total_numel = c.space->total_numel();
        out->fingerprint = c.space->fingerprint();
        return RS_OK;
    });
}

int rs_plan_dump(const rs_plan_t* p, int device, char** out, size_t* len) {
    return guarded([&] {
        *out = dup_string(device >= 0 ? core::dump(p->core, gpuplan::box_routes_gpu(p->core, device, nullptr), expand(p, device))
                                      : core::dump(p->core, expand(p, device)),
                          len);
        return RS_OK;
    });
}

int rs_plan_validate(const rs_plan_t* p, int64_t drop, char** report, size_t* len, int64_t* n_violations) {
    return guarded([&] {
        const std::vector<std::string> v = core::validate_plan(p->core, core::expand_flat_host(p->core), drop);
        std::string s;
        for (const std::string& x : v) s += x + "\n";
        *n_violations = static_cast<int64_t>(v.size());
        *report = dup_string(s, len);
        return RS_OK;
    });
}

int rs_plan_expand_timed(const rs_plan_t* p, int device, double* ms, int64_t* n_runs) {
    return guarded([&] {
        double t = 0;
        std::vector<core::FlatXfer> v;
        if (device >= 0) {
            v = gpuplan::expand_flat_gpu(p->core, device, &t);
        } else {
            const auto t0 = std::chrono::steady_clock::now();
            v = core::expand_flat_host(p->core);
            t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
        *ms = t;
        *n_runs = static_cast<int64_t>(v.size());
        return RS_OK;
    });
}

int rs_plan_box_routes_timed(const rs_plan_t* p, int device, double* ms, int64_t* n_boxes, int* equal_host) {
    return guarded([&] {
        double t = 0;
        const std::vector<core::BoxXfer> v = gpuplan::box_routes_gpu(p->core, device, &t);
        *ms = t;
        *n_boxes = static_cast<int64_t>(v.size());
        bool eq = v.size() == p->core.box.size();
        for (size_t i = 0; eq && i < v.size(); ++i) {
            const core::BoxXfer &a = v[i], &b = p->core.box[i];
            eq = a.kind == b.kind && a.tensor == b.tensor && a.src == b.src && a.dst == b.dst && a.count == b.count &&
                 a.bytes == b.bytes && std::equal(a.lo, a.lo + 4, b.lo) && std::equal(a.hi, a.hi + 4, b.hi);
        }
        *equal_host = eq ? 1 : 0;
        return RS_OK;
    });
}

int rs_plan_dump_rows_host(const rs_plan_t* p, char** out, size_t* len) {
    return guarded([&] {
        *out = dup_string(core::dump(p->core, core::expand_flat_rows_host(p->core)), len);
        return RS_OK;
    });
}

int rs_plan_transfers(const rs_plan_t* p, int device, rs_transfer_t** out, int64_t* n) {
    return guarded([&] {
        const core::PlanCore& c = p->core;
        const std::vector<core::FlatXfer> flat = expand(p, device);
        // device >= 0: both planner halves on the GPU (box intersections + ZeRO runs)
        const std::vector<core::BoxXfer> boxes = device >= 0 ? gpuplan::box_routes_gpu(c, device, nullptr) : c.box;
        const size_t total = boxes.size() + flat.size();
        rs_transfer_t* arr = static_cast<rs_transfer_t*>(std::calloc(total ? total : 1, sizeof(rs_transfer_t)));
        if (!arr) throw std::bad_alloc();
        size_t bi = 0, fi = 0, k = 0;
        while (bi < boxes.size() || fi < flat.size()) {
            bool take_box;
            if (bi == boxes.size()) take_box = false;
            else if (fi == flat.size()) take_box = true;
            else {
                const auto& b = boxes[bi];
                const auto& f = flat[fi];
                take_box = b.src != f.src ? b.src < f.src : b.dst != f.dst ? b.dst < f.dst : b.kind < 1;
            }
            rs_transfer_t& t = arr[k++];
            if (take_box) {
                const auto& b = boxes[bi++];
                t.kind = b.kind;
                t.tensor = b.tensor;
                t.flat = 0;
                t.ndim = static_cast<int>(c.space->entries()[static_cast<size_t>(b.tensor)].spec.shape.size());
                for (int d = 0; d < 4; ++d) t.lo[d] = b.lo[d], t.hi[d] = b.hi[d];
                t.src_rank = b.src;
                t.dst_rank = b.dst;
                t.count = b.count;
                t.bytes = b.bytes;
            } else {
                const auto& f = flat[fi++];
                t.kind = RS_KIND_OPTIM;
                t.tensor = -1;
                t.flat = 1;
                t.ndim = 1;
                t.lo[0] = f.lo;
                t.hi[0] = f.hi;
                t.src_rank = f.src;
                t.dst_rank = f.dst;
                t.count = f.hi - f.lo;
                t.bytes = t.count * kOptimStateBytes;
            }
            t.src_phys = c.wm.src_phys[static_cast<size_t>(t.src_rank)];
            t.dst_phys = c.wm.dst_phys[static_cast<size_t>(t.dst_rank)];
        }
        *out = arr;
        *n = static_cast<int64_t>(total);
        return RS_OK;
    });
}

namespace {
const core::RankGeom& rank_geom(const rs_plan_t* p, int side, int rank) {
    if (side != RS_SIDE_SRC && side != RS_SIDE_DST) throw ConfigError("bad side");
    const core::Side& S = side == RS_SIDE_SRC ? p->core.src : p->core.dst;
    if (rank < 0 || rank >= static_cast<int>(S.ranks.size())) throw ConfigError("rank out of range");
    return S.ranks[static_cast<size_t>(rank)];
}
}  // namespace

int rs_plan_rank_geom(const rs_plan_t* p, int side, int rank, rs_rank_geom_t* out) {
    return guarded([&] {
        const core::RankGeom& g = rank_geom(p, side, rank);
        out->phys = g.phys;
        out->n_segments = static_cast<int>(g.segs.size());
        out->dense_len = g.dense_len;
        out->expert_len = g.expert_len;
        out->dshard_lo = g.dshard.lo;
        out->dshard_hi = g.dshard.hi;
        out->eshard_lo = g.eshard.lo;
        out->eshard_hi = g.eshard.hi;
        out->param_bytes = g.param_bytes;
        out->nelem = g.nelem;
        out->optim_len = g.optim_len;
        out->scalar_bytes = p->core.opts.scalar_words * kScalarWordBytes;
        return RS_OK;
    });
}

int rs_plan_segments(const rs_plan_t* p, int side, int rank, rs_segment_t* out, int cap, int* n) {
    return guarded([&] {
        const core::RankGeom& g = rank_geom(p, side, rank);
        *n = static_cast<int>(g.segs.size());
        for (int i = 0; i < *n && i < cap; ++i) {
            const core::Seg& sg = g.segs[static_cast<size_t>(i)];
            rs_segment_t& o = out[i];
            o.tensor = sg.tensor;
            o.expert = sg.expert ? 1 : 0;
            for (int d = 0; d < 4; ++d) o.box_lo[d] = sg.blo[d], o.box_hi[d] = sg.bhi[d];
            o.local_lo = sg.local_lo;
            o.local_hi = sg.local_hi;
            o.param_byte_off = sg.param_byte_off;
            o.elem_off = sg.elem_off;
        }
        return RS_OK;
    });
}

int rs_plan_num_tensors(const rs_plan_t* p, int* n) {
    return guarded([&] {
        *n = p->core.ntensors();
        return RS_OK;
    });
}

int rs_plan_tensor(const rs_plan_t* p, int index, char* id_buf, int cap, int64_t shape[4], int* ndim, int* dtype_bytes) {
    return guarded([&] {
        if (index < 0 || index >= p->core.ntensors()) throw ConfigError("tensor index out of range");
        const TensorSpec& t = p->core.space->entries()[static_cast<size_t>(index)].spec;
        if (cap > 0) {
            const size_t k = std::min(static_cast<size_t>(cap - 1), t.tensor_id.size());
            std::memcpy(id_buf, t.tensor_id.data(), k);
            id_buf[k] = 0;
        }
        *ndim = static_cast<int>(t.shape.size());
        for (int d = 0; d < 4; ++d) shape[d] = d < *ndim ? t.shape[static_cast<size_t>(d)] : 1;
        *dtype_bytes = t.dtype_bytes;
        return RS_OK;
    });
}

int rs_plan_placement(const rs_plan_t* p, int n_gpus, int gpu, rs_placement_stats_t* out) {
    return guarded([&] {
        if (n_gpus < 1 || gpu < 0 || gpu >= n_gpus) throw ConfigError("bad placement");
        const exec::PlacementStats s = exec::placement_stats(p->core, n_gpus, gpu);
        out->local_bytes = s.local_bytes;
        out->out_bytes = s.out_bytes;
        out->in_bytes = s.in_bytes;
        out->ops = s.ops;
        return RS_OK;
    });
}

int rs_plan_traffic(const rs_plan_t* p, int64_t* out, int cap, int* n_phys) {
    return guarded([&] {
        int n = 0;
        const std::vector<std::int64_t> m = exec::traffic_matrix(p->core, &n);
        if (n_phys) *n_phys = n;
        if (out && cap >= n * n) std::copy(m.begin(), m.end(), out);
        return RS_OK;
    });
}

int rs_plan_regions(const rs_plan_t* p, int side, char** out, size_t* len) {
    return guarded([&] {
        const ModelSpace& space = *p->core.space;
        const ParallelConfig& cfg = side == RS_SIDE_SRC ? p->core.src_cfg : p->core.dst_cfg;
        std::string s;
        for (int r = 0; r < cfg.world_size(); ++r) {
            const RegionSet reg = project(space, cfg, r);
            for (const auto& [id, boxes] : reg.boxes)
                for (const Box& b : boxes) s += strfmt("rank %d param %s %s\n", r, id.c_str(), format_box(b).c_str());
            const LocalLayout L = local_layout(space, cfg, r);
            for (const auto& seg : L.dense)
                s += strfmt("rank %d layout dense %s %s %lld %lld\n", r, seg.tensor_id.c_str(), format_box(seg.box).c_str(),
                            static_cast<long long>(seg.local_lo), static_cast<long long>(seg.local_hi));
            for (const auto& seg : L.expert)
                s += strfmt("rank %d layout expert %s %s %lld %lld\n", r, seg.tensor_id.c_str(), format_box(seg.box).c_str(),
                            static_cast<long long>(seg.local_lo), static_cast<long long>(seg.local_hi));
            if (cfg.zero_enabled)
                for (const Interval& iv : project_optimizer(space, cfg, r).flat)
                    s += strfmt("rank %d optim %s\n", r, format_interval(iv).c_str());
        }
        *out = dup_string(s, len);
        return RS_OK;
    });
}

int rs_config_groups(const rs_cfg_t* cfg, int dim, int* out, int cap, int* n_groups, int* group_size) {
    return guarded([&] {
        if (dim < 0 || dim > 4) throw ConfigError("bad group dimension");
        const auto g = parallel_groups(to_cfg(*cfg), static_cast<GroupDim>(dim));
        *n_groups = static_cast<int>(g.size());
        *group_size = g.empty() ? 0 : static_cast<int>(g[0].size());
        int k = 0;
        for (const auto& grp : g)
            for (int r : grp) {
                if (k < cap) out[k] = r;
                ++k;
            }
        return RS_OK;
    });
}

int rs_rank_coord(const rs_cfg_t* cfg, int rank, int coord[5]) {
    return guarded([&] {
        const RankCoord c = rank_coord(to_cfg(*cfg), rank);
        coord[0] = c.pp_rank, coord[1] = c.dp_rank, coord[2] = c.tp_rank, coord[3] = c.ep_rank, coord[4] = c.edp_rank;
        return RS_OK;
    });
}

int rs_xor_peer(int i, int s, int n) { return sched::xor_peer(i, s, n); }

int rs_memory_aware_chunk(const int* steps, const int64_t* cost, int n_steps, const int64_t* mem_avail, int n_ranks,
                          int* stage_of_step, int64_t* budget) {
    return guarded([&] {
        std::vector<int> st(steps, steps + n_steps);
        int maxs = 0;
        for (int x : st) maxs = std::max(maxs, x);
        std::vector<std::int64_t> c(static_cast<size_t>(maxs) + 1, 0);
        for (int k = 0; k < n_steps; ++k) c[static_cast<size_t>(steps[k])] = cost[k];
        std::int64_t M = 0;
        const auto stages = sched::memory_aware_chunk(st, c, std::vector<std::int64_t>(mem_avail, mem_avail + n_ranks), &M);
        for (size_t g = 0; g < stages.size(); ++g)
            for (int x : stages[g])
                for (int k = 0; k < n_steps; ++k)
                    if (steps[k] == x) stage_of_step[k] = static_cast<int>(g);
        if (budget) *budget = M;
        return RS_OK;
    });
}

int rs_schedule_build(const rs_plan_t* p, const int64_t* mem_avail, int n, int promote, rs_schedule_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto s = std::make_unique<rs_schedule>();
        s->plan = p;
        std::vector<std::int64_t> avail;
        if (mem_avail) avail.assign(mem_avail, mem_avail + n);
        s->T = sched::build_schedule(p->core, core::expand_flat_host(p->core), avail, promote != 0);
        *out = s.release();
        return RS_OK;
    });
}

void rs_schedule_destroy(rs_schedule_t* s) { delete s; }

int rs_schedule_summary(const rs_schedule_t* s, rs_schedule_summary_t* out) {
    return guarded([&] {
        const sched::TransitionSchedule& T = s->T;
        std::memset(out, 0, sizeof *out);
        out->num_devices = T.N;
        out->num_stages = static_cast<int>(T.stages.size());
        out->num_collectives = static_cast<int>(T.collectives.size());
        for (const auto& st : T.stages) out->num_steps += static_cast<int>(st.steps.size());
        out->budget = T.budget;
        std::int64_t total = 0;
        for (const auto& f : T.frags) total += f.bytes;
        for (const auto& c : T.collectives) out->collective_bytes += c.bytes;
        out->p2p_bytes = total - out->collective_bytes;
        out->num_fragments = static_cast<int64_t>(T.frags.size());
        return RS_OK;
    });
}

int rs_schedule_stage(const rs_schedule_t* s, int k, int* steps, int cap, int* n, int64_t* mem_cost) {
    return guarded([&] {
        const auto& st = s->T.stages.at(static_cast<size_t>(k));
        *n = static_cast<int>(st.steps.size());
        for (int i = 0; i < *n && i < cap; ++i) steps[i] = st.steps[static_cast<size_t>(i)];
        if (mem_cost) *mem_cost = st.mem_cost;
        return RS_OK;
    });
}

int rs_schedule_peer(const rs_schedule_t* s, int k, int q, int dev, int* peer, int64_t* send_bytes, int64_t* recv_bytes) {
    return guarded([&] {
        const auto& rs = s->T.stages.at(static_cast<size_t>(k)).ranks.at(static_cast<size_t>(dev)).at(static_cast<size_t>(q));
        *peer = rs.peer;
        *send_bytes = rs.send.bytes;
        *recv_bytes = rs.recv.bytes;
        return RS_OK;
    });
}

int rs_schedule_collective(const rs_schedule_t* s, int c, int* kind, int* root, int64_t* bytes, int* participants, int cap,
                           int* n) {
    return guarded([&] {
        const auto& op = s->T.collectives.at(static_cast<size_t>(c));
        *kind = static_cast<int>(op.kind);
        *root = op.root;
        *bytes = op.bytes;
        *n = static_cast<int>(op.participants.size());
        for (int i = 0; i < *n && i < cap; ++i) participants[i] = op.participants[static_cast<size_t>(i)];
        return RS_OK;
    });
}

int rs_schedule_dump(const rs_schedule_t* s, char** out, size_t* len) {
    return guarded([&] {
        *out = dup_string(sched::dump_schedule(s->plan->core, s->T), len);
        return RS_OK;
    });
}

int rs_execute(const rs_plan_t* p, const rs_exec_opts_t* o, const rs_state_buffer_t* bufs, int n_bufs, void* stream,
               int mode, int* launches) {
    return guarded([&] {
        if (mode != RS_EXEC_FUSED) throw ConfigError("rs_execute: bad mode");
        rs_exec_t* e = nullptr;
        const int rc = rs_exec_create(p, o, &e);
        if (rc != RS_OK) return rc;
        std::unique_ptr<rs_exec_t, void (*)(rs_exec_t*)> guard(e, rs_exec_destroy);
        for (int i = 0; i < n_bufs; ++i)
            e->ex->bind(bufs[i].side, bufs[i].rank, bufs[i].buf, bufs[i].ptr, bufs[i].bytes);
        e->ex->prepare();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int n = e->ex->run(st);
        if (cudaStreamSynchronize(st) != cudaSuccess) throw exec::CudaError("rs_execute: stream failed");
        if (launches) *launches = n;
        return RS_OK;
    });
}

int rs_exec_create(const rs_plan_t* p, const rs_exec_opts_t* o, rs_exec_t** out) {
    return guarded([&] {
        *out = nullptr;
        exec::ExecConfig cfg;
        if (o) {
            cfg.n_gpus = o->n_gpus;
            cfg.gpu = o->gpu;
            cfg.device = o->device;
            cfg.with_grads = o->with_grads != 0;
            cfg.tile_bytes = o->tile_bytes;
            cfg.ctas_per_sm = o->ctas_per_sm;
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw exec::CudaError("no CUDA device: the executor has no CPU fallback");
        auto e = std::make_unique<rs_exec>();
        e->plan = p;
        e->ex = std::make_unique<exec::Executor>(p->core, cfg);
        *out = e.release();
        return RS_OK;
    });
}

void rs_exec_destroy(rs_exec_t* e) { delete e; }

int rs_exec_alloc(rs_exec_t* e) {
    return guarded([&] {
        e->ex->alloc();
        return RS_OK;
    });
}

int rs_exec_bind(rs_exec_t* e, int side, int rank, int buf, void* dptr, int64_t bytes) {
    return guarded([&] {
        e->ex->bind(side, rank, buf, dptr, bytes);
        return RS_OK;
    });
}

int rs_exec_buffer(rs_exec_t* e, int side, int rank, int buf, void** dptr, int64_t* bytes, int* gpu) {
    return guarded([&] {
        if (side < 0 || side > 1 || buf < 0 || buf >= exec::kNumBufs) throw ConfigError("bad buffer id");
        const int n = side == 0 ? e->plan->core.src_cfg.world_size() : e->plan->core.dst_cfg.world_size();
        if (rank < 0 || rank >= n) throw ConfigError("bad rank");
        std::int64_t b = 0;
        *dptr = e->ex->buffer(side, rank, buf, &b);
        *bytes = b;
        if (gpu) *gpu = e->ex->rank_gpu(side, rank);
        return RS_OK;
    });
}

int rs_exec_ipc_export(rs_exec_t* e, void* out, size_t cap, size_t* len) {
    return guarded([&] {
        const std::vector<std::uint8_t> blob = e->ex->export_ipc();
        *len = blob.size();
        if (out && cap >= blob.size()) std::memcpy(out, blob.data(), blob.size());
        else if (out) throw ConfigError("ipc export buffer too small");
        return RS_OK;
    });
}

int rs_exec_ipc_import(rs_exec_t* e, const void* blob, size_t len) {
    return guarded([&] {
        e->ex->import_ipc(static_cast<const std::uint8_t*>(blob), len);
        return RS_OK;
    });
}

int rs_exec_prepare(rs_exec_t* e) {
    return guarded([&] {
        e->ex->prepare();
        return RS_OK;
    });
}

int rs_exec_prepare_staged(rs_exec_t* e) {
    return guarded([&] {
        e->ex->prepare(true);
        return RS_OK;
    });
}

int rs_sync_create(int rank, int world, int device, rs_sync_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto s = std::make_unique<rs_sync>();
        s->b = std::make_unique<sync::DeviceBarrier>(rank, world, device);
        *out = s.release();
        return RS_OK;
    });
}

void rs_sync_destroy(rs_sync_t* s) { delete s; }

int rs_sync_export(const rs_sync_t* s, void* out, size_t cap, size_t* len) {
    return guarded([&] {
        const std::vector<std::uint8_t> v = s->b->export_handle();
        *len = v.size();
        if (out && cap >= v.size()) std::memcpy(out, v.data(), v.size());
        return RS_OK;
    });
}

int rs_sync_import(rs_sync_t* s, int peer, const void* blob, size_t len) {
    return guarded([&] {
        s->b->import_handle(peer, static_cast<const std::uint8_t*>(blob), len);
        return RS_OK;
    });
}

int rs_sync_barrier(rs_sync_t* s, void* stream) {
    return guarded([&] {
        s->b->arrive_and_wait(static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_sync_status(rs_sync_t* s, int* timed_out) {
    return guarded([&] {
        *timed_out = s->b->status();
        return RS_OK;
    });
}

int rs_exec_set_plan(rs_exec_t* e, const rs_plan_t* p) {
    return guarded([&] {
        e->ex->set_plan(p->core);
        e->plan = p;
        return RS_OK;
    });
}

int rs_exec_set_collectives(rs_exec_t* e, int on) {
    return guarded([&] {
        e->ex->set_collectives(on != 0);
        return RS_OK;
    });
}

int rs_exec_gpu_of_phys(const rs_exec_t* e, int phys, int* gpu) {
    return guarded([&] {
        *gpu = e->ex->gpu_of_phys(phys);
        return RS_OK;
    });
}

int rs_plan_participants(const rs_plan_t* p, int* phys, int cap, int* n) {
    return guarded([&] {
        const auto& r = p->core.routes;
        *n = static_cast<int>(r.size());
        for (int i = 0; i < *n && i < cap; ++i) phys[i] = r[static_cast<size_t>(i)].phys;
        return RS_OK;
    });
}

int rs_exec_channel_bytes(const rs_exec_t* e, int src_phys, int dst_phys, int64_t* bytes) {
    return guarded([&] {
        *bytes = e->ex->channel_bytes(src_phys, dst_phys);
        return RS_OK;
    });
}

int rs_exec_channel_ops(const rs_exec_t* e, int src_phys, int dst_phys, int64_t* sizes, int64_t cap, int64_t* n) {
    return guarded([&] {
        const std::vector<std::int64_t> v = e->ex->channel_ops(src_phys, dst_phys);
        *n = static_cast<int64_t>(v.size());
        for (int64_t i = 0; i < *n && i < cap; ++i) sizes[i] = v[static_cast<size_t>(i)];
        return RS_OK;
    });
}

int rs_exec_pack(rs_exec_t* e, int src_phys, int dst_phys, void* dbuf, void* stream) {
    return guarded([&] {
        e->ex->pack(src_phys, dst_phys, dbuf, static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_exec_unpack(rs_exec_t* e, int src_phys, int dst_phys, const void* dbuf, void* stream) {
    return guarded([&] {
        e->ex->unpack(src_phys, dst_phys, dbuf, static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_exec_fill(rs_exec_t* e, int side, uint64_t seed, void* stream) {
    return guarded([&] {
        e->ex->fill(side, seed, static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_exec_run(rs_exec_t* e, void* stream, int* launches) {
    return guarded([&] {
        const int n = e->ex->run(static_cast<cudaStream_t>(stream));
        if (launches) *launches = n;
        return RS_OK;
    });
}

int rs_exec_verify(rs_exec_t* e, int side, uint64_t seed, void* stream, int64_t* mismatches, int64_t* first_bad) {
    return guarded([&] {
        std::int64_t fb = -1;
        const std::int64_t bad = e->ex->verify(side, seed, static_cast<cudaStream_t>(stream), &fb);
        if (mismatches) *mismatches = bad;
        if (first_bad) *first_bad = fb;
        return bad ? fail(RS_ERR_VIOLATION, strfmt("%lld mismatching elements (first flat index %lld)",
                                                   static_cast<long long>(bad), static_cast<long long>(fb)))
                   : RS_OK;
    });
}

int rs_enable_peer_access(int device, int peer) {
    return guarded([&] {
        if (cudaSetDevice(device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
        const cudaError_t r = cudaDeviceEnablePeerAccess(peer, 0);
        if (r == cudaErrorPeerAccessAlreadyEnabled) {
            cudaGetLastError();
        } else if (r != cudaSuccess) {
            throw exec::CudaError(strfmt("cudaDeviceEnablePeerAccess(%d -> %d): %s", device, peer, cudaGetErrorString(r)));
        }
        return RS_OK;
    });
}

int rs_exec_read(rs_exec_t* e, int side, int rank, int buf, int64_t offset, void* host, int64_t bytes, void* stream) {
    return guarded([&] {
        if (side < 0 || side > 1 || buf < 0 || buf >= exec::kNumBufs) throw ConfigError("bad buffer id");
        std::int64_t n = 0;
        void* p = e->ex->buffer(side, rank, buf, &n);
        if (!p || offset < 0 || bytes < 0 || offset + bytes > n) throw ConfigError("read outside the buffer");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (cudaMemcpyAsync(host, static_cast<const char*>(p) + offset, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost,
                            st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            throw exec::CudaError("rs_exec_read: copy failed");
        return RS_OK;
    });
}

int rs_exec_stats(const rs_exec_t* e, rs_exec_stats_t* out) {
    return guarded([&] {
        const exec::ExecStats& s = e->ex->stats();
        out->local_bytes = s.local_bytes;
        out->remote_bytes = s.remote_bytes;
        out->tiles = s.tiles;
        for (int i = 0; i < 5; ++i) out->tiles_by_class[i] = s.tiles_by_class[i];
        out->launches = s.launches;
        out->mc_bytes = s.mc_bytes;
        out->dup_bytes = s.dup_bytes;
        out->scatter_bytes = s.scatter_bytes;
        out->gather_bytes = s.gather_bytes;
        return RS_OK;
    });
}

int rs_exec_run_graph(rs_exec_t* e, void* stream, int* launches) {
    return guarded([&] {
        *launches = e->ex->run_graph(static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_exec_set_stages(rs_exec_t* e, const int* dst_order, int n) {
    return guarded([&] {
        e->ex->set_stage_order(std::vector<int>(dst_order, dst_order + (dst_order ? n : 0)));
        return RS_OK;
    });
}

int rs_exec_set_stage_groups(rs_exec_t* e, const int* dst_order, const int* cuts, int n) {
    return guarded([&] {
        e->ex->set_stage_order(std::vector<int>(dst_order, dst_order + n),
                               cuts ? std::vector<int>(cuts, cuts + n) : std::vector<int>());
        return RS_OK;
    });
}

int rs_arena_stage_cuts(const rs_arena_t* a, int dir, int* out, int cap, int* n) {
    return guarded([&] {
        if (dir < 0 || dir > 1) throw ConfigError("bad direction");
        const std::vector<int>& c = a->a->stage_cuts(dir);
        *n = static_cast<int>(c.size());
        for (int i = 0; i < *n && i < cap; ++i) out[i] = c[static_cast<size_t>(i)];
        return RS_OK;
    });
}

int rs_arena_create(const rs_plan_t* ab, const rs_plan_t* ba, int device, int64_t cap_bytes, int64_t chunk_bytes,
                    int with_grads, rs_arena_t** out) {
    return guarded([&] {
        *out = nullptr;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw exec::CudaError("no CUDA device");
        mem::ArenaConfig cfg;
        cfg.device = device;
        cfg.cap_bytes = cap_bytes;
        if (chunk_bytes > 0) cfg.chunk_bytes = chunk_bytes;
        auto a = std::make_unique<rs_arena>();
        a->a = std::make_unique<mem::Arena>(ab->core, ba ? &ba->core : nullptr, cfg, with_grads != 0);
        *out = a.release();
        return RS_OK;
    });
}

void rs_arena_destroy(rs_arena_t* a) { delete a; }

int rs_arena_create_multi(const rs_plan_t* ab, const rs_plan_t* ba, int n_gpus, int gpu, int device, int64_t cap_bytes,
                          int64_t chunk_bytes, int with_grads, int groups, int bands, rs_arena_t** out) {
    return guarded([&] {
        *out = nullptr;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw exec::CudaError("no CUDA device");
        if (n_gpus < 1 || gpu < 0 || gpu >= n_gpus) throw ConfigError("bad arena placement");
        mem::ArenaConfig cfg;
        cfg.device = device;
        cfg.cap_bytes = cap_bytes;
        if (chunk_bytes > 0) cfg.chunk_bytes = chunk_bytes;
        cfg.groups = groups;
        cfg.bands = bands;
        auto a = std::make_unique<rs_arena>();
        a->a = std::make_unique<mem::Arena>(ab->core, ba ? &ba->core : nullptr, cfg, with_grads != 0, n_gpus, gpu);
        *out = a.release();
        return RS_OK;
    });
}

int rs_arena_export(const rs_arena_t* a, int** fds, int* n_fds, void** table, size_t* table_len) {
    return guarded([&] {
        std::vector<int> f;
        std::vector<std::uint8_t> t;
        a->a->export_local(&f, &t);
        *fds = static_cast<int*>(std::malloc(sizeof(int) * (f.empty() ? 1 : f.size())));
        *table = std::malloc(t.empty() ? 1 : t.size());
        if (!*fds || !*table) throw std::bad_alloc();
        std::memcpy(*fds, f.data(), sizeof(int) * f.size());
        std::memcpy(*table, t.data(), t.size());
        *n_fds = static_cast<int>(f.size());
        *table_len = t.size();
        return RS_OK;
    });
}

int rs_arena_import(rs_arena_t* a, const int* fds, int n_fds, const void* table, size_t table_len) {
    return guarded([&] {
        const auto* t = static_cast<const std::uint8_t*>(table);
        a->a->import_peer(std::vector<int>(fds, fds + n_fds), std::vector<std::uint8_t>(t, t + table_len));
        return RS_OK;
    });
}

int rs_fdx_listen(const char* name, int* sock) {
    return guarded([&] {
        *sock = fdx::listen_on(name);
        return RS_OK;
    });
}

int rs_fdx_send(const char* peer_name, const int* fds, int n_fds, const void* payload, size_t len) {
    return guarded([&] {
        const auto* p = static_cast<const std::uint8_t*>(payload);
        fdx::send_fds(peer_name, std::vector<int>(fds, fds + n_fds), std::vector<std::uint8_t>(p, p + len));
        return RS_OK;
    });
}

int rs_fdx_recv(int sock, int** fds, int* n_fds, void** payload, size_t* len) {
    return guarded([&] {
        std::vector<std::uint8_t> pl;
        const std::vector<int> f = fdx::recv_fds(sock, &pl);
        *fds = static_cast<int*>(std::malloc(sizeof(int) * (f.empty() ? 1 : f.size())));
        *payload = std::malloc(pl.empty() ? 1 : pl.size());
        if (!*fds || !*payload) throw std::bad_alloc();
        std::memcpy(*fds, f.data(), sizeof(int) * f.size());
        std::memcpy(*payload, pl.data(), pl.size());
        *n_fds = static_cast<int>(f.size());
        *len = pl.size();
        return RS_OK;
    });
}

int rs_fdx_close(int fd) {
    fdx::close_fd(fd);
    return RS_OK;
}

int rs_exec_num_stages(const rs_exec_t* e, int* n) {
    return guarded([&] {
        *n = e->ex->num_stages();
        return RS_OK;
    });
}

int rs_exec_run_stage(rs_exec_t* e, int stage, void* stream, int* launches) {
    return guarded([&] {
        const int k = e->ex->run_stage(stage, static_cast<cudaStream_t>(stream));
        if (launches) *launches = k;
        return RS_OK;
    });
}

int rs_arena_buffer(const rs_arena_t* a, int layout, int rank, int buf, void** dptr, int64_t* bytes) {
    return guarded([&] {
        if (layout < 0 || layout > 1 || buf < 0 || buf >= exec::kNumBufs) throw ConfigError("bad buffer id");
        *dptr = a->a->ptr(layout, rank, buf);
        *bytes = a->a->bytes(layout, rank, buf);
        return RS_OK;
    });
}

int rs_arena_stage_order(const rs_arena_t* a, int dir, int* out, int cap, int* n) {
    return guarded([&] {
        if (dir < 0 || dir > 1) throw ConfigError("bad direction");
        const std::vector<int>& o = a->a->stage_order(dir);
        *n = static_cast<int>(o.size());
        for (int i = 0; i < *n && i < cap; ++i) out[i] = o[static_cast<size_t>(i)];
        return RS_OK;
    });
}

int rs_memory_min_groups(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, int n_gpus,
                         int gpu, int64_t cap_bytes, int* groups, int64_t* physical_bytes) {
    return guarded([&] {
        if (n_gpus < 1 || gpu < 0 || gpu >= n_gpus) throw ConfigError("bad arena placement");
        *groups = mem::min_stage_groups(ab->core, ba ? &ba->core : nullptr, chunk_bytes > 0 ? chunk_bytes : (32ll << 20),
                                        with_grads != 0, n_gpus, gpu, cap_bytes, physical_bytes);
        return RS_OK;
    });
}

int rs_memory_schedule(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, int n_gpus,
                       int gpu, int64_t cap_bytes, int* level, int64_t* physical_bytes) {
    return guarded([&] {
        if (n_gpus < 1 || gpu < 0 || gpu >= n_gpus) throw ConfigError("bad arena placement");
        *level = mem::choose_schedule(ab->core, ba ? &ba->core : nullptr, chunk_bytes > 0 ? chunk_bytes : (32ll << 20),
                                      with_grads != 0, n_gpus, gpu, cap_bytes, physical_bytes);
        return RS_OK;
    });
}

int rs_memory_schedule_costs(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, int n_gpus,
                             int gpu, int64_t* bytes, double* seconds, int cap, int* n) {
    return guarded([&] {
        if (n_gpus < 1 || gpu < 0 || gpu >= n_gpus) throw ConfigError("bad arena placement");
        const auto f = mem::schedule_costs(ab->core, ba ? &ba->core : nullptr, chunk_bytes > 0 ? chunk_bytes : (32ll << 20),
                                           with_grads != 0, n_gpus, gpu);
        *n = static_cast<int>(f.size());
        for (int i = 0; i < *n && i < cap; ++i) {
            bytes[i] = f[static_cast<size_t>(i)].first;
            seconds[i] = f[static_cast<size_t>(i)].second;
        }
        return RS_OK;
    });
}

int rs_memory_schedule_footprints(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, int n_gpus,
                                  int gpu, int64_t* out, int cap, int* n) {
    return guarded([&] {
        if (n_gpus < 1 || gpu < 0 || gpu >= n_gpus) throw ConfigError("bad arena placement");
        const std::vector<std::int64_t> f =
            mem::schedule_footprints(ab->core, ba ? &ba->core : nullptr, chunk_bytes > 0 ? chunk_bytes : (32ll << 20),
                                     with_grads != 0, n_gpus, gpu);
        *n = static_cast<int>(f.size());
        for (int i = 0; i < *n && i < cap; ++i) out[i] = f[static_cast<size_t>(i)];
        return RS_OK;
    });
}

int rs_memory_schedule_level(const rs_plan_t* ab, int n_gpus, int level, int* bands, int* groups) {
    return guarded([&] {
        const std::vector<mem::ScheduleLevel> L = mem::schedule_levels(ab->core, n_gpus);
        if (level < 0 || level >= static_cast<int>(L.size())) throw ConfigError("schedule level out of range");
        *bands = L[static_cast<size_t>(level)].bands;
        *groups = L[static_cast<size_t>(level)].groups;
        return RS_OK;
    });
}

int rs_memory_plan_ex(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, int n_gpus, int gpu,
                      int groups, int bands, rs_arena_stats_t* stats, int64_t* violations, int* order_ab, int* order_ba,
                      int cap) {
    return guarded([&] {
        const mem::MemoryPlan mp = mem::plan_memory(ab->core, ba ? &ba->core : nullptr,
                                                    chunk_bytes > 0 ? chunk_bytes : (32ll << 20), with_grads != 0,
                                                    n_gpus, gpu, groups, bands);
        stats->bands = mp.bands;
        stats->physical_bytes = mp.stats.physical_bytes;
        stats->a_bytes = mp.stats.a_bytes;
        stats->b_bytes = mp.stats.b_bytes;
        stats->aliased_bytes = mp.stats.aliased_bytes;
        stats->chunks = mp.stats.chunks;
        *violations = mem::simulate_memory_plan(mp, ab->core, ba ? &ba->core : nullptr);
        stats->stage_groups[0] = stats->stage_groups[1] = 0;
        for (int d = 0; d < 2; ++d)
            for (int c : mp.cut[d]) stats->stage_groups[d] += c;
        for (int d = 0; d < 2; ++d) {
            int* o = d == 0 ? order_ab : order_ba;
            if (!o) continue;
            for (int i = 0; i < cap; ++i) o[i] = i < static_cast<int>(mp.order[d].size()) ? mp.order[d][static_cast<size_t>(i)] : -1;
        }
        return RS_OK;
    });
}

int rs_memory_plan_cuts(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, int n_gpus, int gpu,
                        int groups, int bands, int dir, int* cuts, int cap, int* n) {
    return guarded([&] {
        if (dir < 0 || dir > 1) throw ConfigError("bad direction");
        const mem::MemoryPlan mp = mem::plan_memory(ab->core, ba ? &ba->core : nullptr,
                                                    chunk_bytes > 0 ? chunk_bytes : (32ll << 20), with_grads != 0,
                                                    n_gpus, gpu, groups, bands);
        const std::vector<int>& c = mp.cut[dir];
        *n = static_cast<int>(c.size());
        for (int i = 0; i < *n && i < cap; ++i) cuts[i] = c[static_cast<size_t>(i)];
        return RS_OK;
    });
}

int rs_memory_plan(const rs_plan_t* ab, const rs_plan_t* ba, int64_t chunk_bytes, int with_grads, rs_arena_stats_t* stats,
                   int64_t* violations, int* order_ab, int* order_ba, int cap) {
    return rs_memory_plan_ex(ab, ba, chunk_bytes, with_grads, 1, 0, 0, 1, stats, violations, order_ab, order_ba, cap);
}

int rs_arena_release_through(rs_arena_t* a, int stage, int64_t* freed) {
    return guarded([&] {
        *freed = a->a->release_through(stage);
        return RS_OK;
    });
}

int rs_arena_stats(const rs_arena_t* a, rs_arena_stats_t* out) {
    return guarded([&] {
        const mem::ArenaStats& s = a->a->stats();
        out->physical_bytes = s.physical_bytes;
        out->a_bytes = s.a_bytes;
        out->b_bytes = s.b_bytes;
        out->aliased_bytes = s.aliased_bytes;
        out->bands = a->a->bands();
        out->chunks = s.chunks;
        for (int d = 0; d < 2; ++d) {
            out->stage_groups[d] = 0;
            for (int c : a->a->stage_cuts(d)) out->stage_groups[d] += c;
        }
        return RS_OK;
    });
}


struct rs_mc {
    std::unique_ptr<mem::Multicast> m;
};

int rs_exec_bcast_groups(rs_exec_t* e, rs_bcast_group_t* out, int cap, int* n) {
    return guarded([&] {
        const std::vector<exec::BcastGroup>& G = e->ex->bcast_groups();
        *n = static_cast<int>(G.size());
        for (int i = 0; i < *n && i < cap; ++i) {
            const exec::BcastGroup& g = G[static_cast<size_t>(i)];
            rs_bcast_group_t& o = out[i];
            o.id = g.id;
            o.root_rank = g.root_rank;
            o.root_gpu = g.root_gpu;
            o.buf = g.buf;
            o.slot = g.slot;
            if (g.member_ranks.size() > RS_MAX_MEMBERS) throw ConfigError("broadcast group exceeds RS_MAX_MEMBERS");
            o.n_members = static_cast<int>(g.member_ranks.size());
            for (int k = 0; k < o.n_members; ++k) {
                o.member_gpu[k] = g.member_gpus[static_cast<size_t>(k)];
                o.member_rank[k] = g.member_ranks[static_cast<size_t>(k)];
            }
            o.buffer_bytes = g.buffer_bytes;
            o.payload_bytes = g.payload_bytes;
        }
        return RS_OK;
    });
}

int rs_exec_set_multicast(rs_exec_t* e, int id, void* mc_va) {
    return guarded([&] {
        e->ex->set_multicast(id, mc_va);
        return RS_OK;
    });
}

int rs_exec_set_replica_dedup(rs_exec_t* e, int on) {
    return guarded([&] {
        e->ex->set_replica_dedup(on != 0, on == 2);
        return RS_OK;
    });
}

int rs_exec_run_dup(rs_exec_t* e, void* stream, int* launches) {
    return guarded([&] {
        *launches = e->ex->run_dup(static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_mc_create(int64_t bytes, int n_devices, rs_mc_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto m = std::make_unique<rs_mc>();
        m->m = std::make_unique<mem::Multicast>(bytes, n_devices);
        *out = m.release();
        return RS_OK;
    });
}

int rs_mc_import(int fd, int64_t bytes, rs_mc_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto m = std::make_unique<rs_mc>();
        m->m = std::make_unique<mem::Multicast>(fd, bytes);
        *out = m.release();
        return RS_OK;
    });
}

int rs_mc_export(const rs_mc_t* m, int* fd) {
    return guarded([&] {
        *fd = m->m->export_fd();
        return RS_OK;
    });
}

int rs_mc_add_device(rs_mc_t* m, int device) {
    return guarded([&] {
        m->m->add_device(device);
        return RS_OK;
    });
}

int rs_mc_bind_arena(rs_mc_t* m, const rs_arena_t* a, int layout, int rank, int buf) {
    return guarded([&] {
        if (layout < 0 || layout > 1 || buf < 0 || buf >= exec::kNumBufs) throw ConfigError("bad buffer id");
        a->a->bind_multicast(*m->m, layout, rank, buf);
        return RS_OK;
    });
}

int rs_mc_map(rs_mc_t* m, int device, void** mc_va) {
    return guarded([&] {
        *mc_va = m->m->map(device);
        return RS_OK;
    });
}

void rs_mc_destroy(rs_mc_t* m) { delete m; }

struct rs_vmm {
    std::unique_ptr<mem::VmmBuffer> v;
};

int rs_vmm_alloc(int device, int64_t bytes, rs_vmm_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto v = std::make_unique<rs_vmm>();
        v->v = std::make_unique<mem::VmmBuffer>(device, bytes);
        *out = v.release();
        return RS_OK;
    });
}

int rs_vmm_import(int fd, int64_t bytes, int device, rs_vmm_t** out) {
    return guarded([&] {
        *out = nullptr;
        auto v = std::make_unique<rs_vmm>();
        v->v = std::make_unique<mem::VmmBuffer>(fd, bytes, device);
        *out = v.release();
        return RS_OK;
    });
}

int rs_vmm_export(const rs_vmm_t* v, int* fd) {
    return guarded([&] {
        *fd = v->v->export_fd();
        return RS_OK;
    });
}

int rs_vmm_ptr(const rs_vmm_t* v, void** ptr, int64_t* mapped_bytes) {
    return guarded([&] {
        *ptr = v->v->ptr();
        *mapped_bytes = v->v->mapped_bytes();
        return RS_OK;
    });
}

void rs_vmm_free(rs_vmm_t* v) { delete v; }

int rs_mc_bind_vmm(rs_mc_t* m, const rs_vmm_t* v, int64_t mc_offset) {
    return guarded([&] {
        m->m->bind(*v->v, mc_offset);
        return RS_OK;
    });
}

int rs_arena_bind_size(const rs_arena_t* a, int layout, int rank, int buf, int64_t* bytes) {
    return guarded([&] {
        if (layout < 0 || layout > 1 || buf < 0 || buf >= exec::kNumBufs) throw ConfigError("bad buffer id");
        *bytes = a->a->bind_size(layout, rank, buf);
        return RS_OK;
    });
}

struct rs_edm {
    edm::Manager m;
    edm::CommCache comms;
};

namespace {
std::string comm_key(const rs_cfg_t* c) {
    return strfmt("dp%d.tp%d.pp%d.ep%d.z%d.%s", c->dp, c->tp, c->pp, c->ep, c->zero, c->order ? c->order : "pp-dp-tp");
}
}  // namespace

int rs_nccl_unique_id(void* out, size_t cap) {
    return guarded([&] {
        if (cap < edm::kNcclIdBytes) throw ConfigError("rs_nccl_unique_id: buffer smaller than 128 bytes");
        edm::nccl_unique_id(static_cast<std::uint8_t*>(out));
        return RS_OK;
    });
}

int rs_nccl_version(char* out, size_t cap) {
    return guarded([&] {
        const std::string v = edm::nccl_version();
        if (cap) {
            std::strncpy(out, v.c_str(), cap - 1);
            out[cap - 1] = 0;
        }
        return RS_OK;
    });
}

int rs_edm_comm_create(rs_edm_t* e, const rs_cfg_t* cfg, const void* uid, int nranks, int rank, int device,
                       const int colors[5], int* cache_hit, double* init_s, double* split_s) {
    return guarded([&] {
        bool hit = false;
        const edm::CommSet& s = e->comms.get_or_create(comm_key(cfg), static_cast<const std::uint8_t*>(uid), nranks,
                                                       rank, device, colors, &hit);
        if (cache_hit) *cache_hit = hit ? 1 : 0;
        if (init_s) *init_s = hit ? 0.0 : s.init_s;
        if (split_s) *split_s = hit ? 0.0 : s.split_s;
        return RS_OK;
    });
}

int rs_edm_comm_get(rs_edm_t* e, const rs_cfg_t* cfg, int dim, void** comm) {
    return guarded([&] {
        const edm::CommSet* s = e->comms.find(comm_key(cfg));
        *comm = !s ? nullptr : dim < 0 ? s->world : dim < edm::kCommDims ? s->dims[dim] : nullptr;
        return RS_OK;
    });
}

int rs_edm_comm_check(rs_edm_t* e, const rs_cfg_t* cfg, int dim, void* stream, float* sum) {
    return guarded([&] {
        *sum = e->comms.check_allreduce(comm_key(cfg), dim, static_cast<cudaStream_t>(stream));
        return RS_OK;
    });
}

int rs_edm_comm_destroy(rs_edm_t* e, const rs_cfg_t* cfg) {
    return guarded([&] {
        e->comms.destroy(comm_key(cfg));
        return RS_OK;
    });
}

int rs_edm_create(rs_edm_t** out) {
    return guarded([&] {
        *out = new rs_edm;
        return RS_OK;
    });
}

void rs_edm_destroy(rs_edm_t* e) { delete e; }

int rs_edm_groups(rs_edm_t* e, const rs_cfg_t* cfg, int dim, int* out, int cap, int* n_groups, int* group_size,
                  int* cache_hit) {
    return guarded([&] {
        if (dim < 0 || dim > 4) throw ConfigError("bad group dimension");
        bool hit = false;
        const auto& g = e->m.groups(to_cfg(*cfg), static_cast<GroupDim>(dim), &hit);
        *n_groups = static_cast<int>(g.size());
        *group_size = g.empty() ? 0 : static_cast<int>(g[0].size());
        *cache_hit = hit ? 1 : 0;
        int k = 0;
        for (const auto& grp : g)
            for (int r : grp) {
                if (k < cap) out[k] = r;
                ++k;
            }
        return RS_OK;
    });
}

int rs_edm_cache_stats(const rs_edm_t* e, int64_t* hits, int64_t* misses, double* creation_s) {
    return guarded([&] {
        std::int64_t h = 0, m = 0;
        e->m.cache_stats(&h, &m, creation_s);
        *hits = h;
        *misses = m;
        return RS_OK;
    });
}

int rs_edm_prepare_async(rs_edm_t* e, int (*build)(void* arg), void* arg) {
    return guarded([&] {
        if (!build) throw ConfigError("edm: no build function");
        e->m.prepare_async(build, arg);
        return RS_OK;
    });
}

int rs_edm_ready(const rs_edm_t* e, int* ready) {
    return guarded([&] {
        *ready = e->m.ready() ? 1 : 0;
        return RS_OK;
    });
}

int rs_edm_wait(rs_edm_t* e, double* init_s, int* build_rc) {
    return guarded([&] {
        *build_rc = e->m.wait(init_s);
        return RS_OK;
    });
}

int rs_edm_accounting(double init_s, double switch_s, double window_s, double train_step_s, int mode,
                      rs_edm_accounting_t* out) {
    return guarded([&] {
        if (mode < 0 || mode > 2) throw ConfigError("bad edm mode");
        const edm::Accounting a = edm::account(init_s, switch_s, window_s, train_step_s, static_cast<edm::Mode>(mode));
        out->init_s = a.init_s;
        out->overlapped_s = a.overlapped_s;
        out->switch_s = a.switch_s;
        out->exposed_s = a.exposed_s;
        out->ratio = a.ratio;
        return RS_OK;
    });
}

}  // extern "C"
