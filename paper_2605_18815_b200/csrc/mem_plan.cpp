// Host side of the memory-aware arena (arena.hpp): stage units and their order, chunk
// lifetimes, the aliasing assignment, concurrency groups, and an independent execution
// simulation that checks it.
#include <algorithm>
#include <limits>
#include <map>

#include "reshard/arena.hpp"
#include "reshard/pool.hpp"

namespace reshard {
namespace mem {

namespace {

constexpr int kNever = std::numeric_limits<int>::max();

struct Extent {
    std::int64_t lo, hi;  // bytes [lo, hi)
};
struct Owner {
    int layout = -1;
    size_t buf = 0, chunk = 0;
};
Extent src_extent(const exec::CopyOp& op) { return {op.src_off, op.src_off + (op.rows - 1) * op.src_pitch + op.row_bytes}; }
Extent dst_extent(const exec::CopyOp& op) { return {op.dst_off, op.dst_off + (op.rows - 1) * op.dst_pitch + op.row_bytes}; }

std::vector<int> positions(const std::vector<int>& order, size_t n) {
    std::vector<int> pos(n, -1);
    for (size_t s = 0; s < order.size(); ++s) pos[static_cast<size_t>(order[s])] = static_cast<int>(s);
    return pos;
}

int gpu_block(const core::PlanCore& P, int n_gpus) {
    int max_phys = 0;
    for (const auto& r : P.routes) max_phys = std::max(max_phys, r.phys);
    return (max_phys + 1 + n_gpus - 1) / n_gpus;
}

}  // namespace

UnitMap::UnitMap(const core::PlanCore& P, int bands) : nb(std::max(1, bands)), nd(P.dst_cfg.world_size()) {
    const auto& ents = P.space->entries();
    const int L = std::max(1, P.space->num_layers());
    nb = std::min(nb, L);
    band_of_tensor.resize(ents.size());
    for (size_t t = 0; t < ents.size(); ++t) band_of_tensor[t] = ents[t].spec.layer * nb / L;
}

/// source pipeline stages a band-interleaved group takes one band from: the source
/// config's pp degree when it divides the band count, else 1
int interleave_stride(const core::PlanCore& P, int nb) {
    const int S = std::max(1, P.src_cfg.pp);
    return nb % S == 0 ? S : 1;
}

namespace {

// One greedy pass over the units. kFreed: the stage freeing the most old bytes anywhere.
// kPeak: among the stages that keep their GPU under the running peak, the one freeing the
// most old bytes on its own GPU, else the lowest peak. kRounds: kPeak restricted to the
// GPUs in turn, so every G consecutive positions hold one unit per GPU (rounds: all links
// busy in every group). kSpread: kPeak, but among the stages under the peak the one on the
// GPU furthest behind (fewest units taken, relative to its total) — a soft form of rounds,
// so merged groups span several GPUs. Returns the order and the modeled peak (max over
// GPUs of live bytes: old data still to be read + new data written so far).
enum PassMode { kFreed = 0, kPeak = 1, kRounds = 2, kSpread = 3 };
std::pair<std::vector<int>, std::int64_t> greedy_pass(const core::PlanCore& P, const std::vector<exec::CopyOp>& ops,
                                                      int bands, int n_gpus, int mode) {
    const bool peak_first = mode != kFreed;
    const UnitMap U(P, bands);
    const int ns = P.src_cfg.world_size(), nd = P.dst_cfg.world_size();
    const int nsu = ns * U.nb, ndu = nd * U.nb;
    const int per = gpu_block(P, std::max(1, n_gpus));
    auto gpu_src = [&](int r) { return P.wm.src_phys[static_cast<size_t>(r)] / per; };
    auto gpu_dst = [&](int r) { return P.wm.dst_phys[static_cast<size_t>(r)] / per; };
    // bytes read from each source unit (what dies with it) and written into each
    // destination unit (what its stage needs), and which source units each stage reads
    std::vector<std::int64_t> w_src(static_cast<size_t>(nsu), 0), w_dst(static_cast<size_t>(ndu), 0);
    std::vector<std::vector<int>> reads(static_cast<size_t>(ndu));
    for (const exec::CopyOp& op : ops) {
        if (op.tensor < 0) continue;  // the scalar blob (a plain allocation) never frees memory
        const int su = U.unit(op.src_side_rank, op.tensor), du = U.unit(op.dst_rank, op.tensor);
        const std::int64_t b = op.rows * op.row_bytes;
        w_src[static_cast<size_t>(su)] += b;
        w_dst[static_cast<size_t>(du)] += b;
        reads[static_cast<size_t>(du)].push_back(su);
    }
    std::vector<int> remaining(static_cast<size_t>(nsu), 0);
    for (auto& v : reads) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        for (int su : v) ++remaining[static_cast<size_t>(su)];
    }
    // per-GPU live bytes (ties: lower unit index, so every rank derives the same order)
    const int G = std::max(1, n_gpus);
    std::vector<std::int64_t> live(static_cast<size_t>(G), 0);
    for (int su = 0; su < nsu; ++su)
        if (remaining[static_cast<size_t>(su)]) live[static_cast<size_t>(gpu_src(su / U.nb))] += w_src[static_cast<size_t>(su)];
    std::int64_t peak = *std::max_element(live.begin(), live.end());
    std::vector<char> done(static_cast<size_t>(ndu), 0);
    std::vector<int> order;
    order.reserve(static_cast<size_t>(ndu));
    std::vector<int> left(static_cast<size_t>(G), 0);
    for (int du = 0; du < ndu; ++du) ++left[static_cast<size_t>(gpu_dst(du / U.nb))];
    const std::vector<int> total_units = left;
    auto progress = [&](int g) {  // fraction of GPU g's units already ordered
        return total_units[static_cast<size_t>(g)]
                   ? 1.0 - static_cast<double>(left[static_cast<size_t>(g)]) / total_units[static_cast<size_t>(g)]
                   : 1.0;
    };
    int turn = 0;
    for (int step = 0; step < ndu; ++step) {
        int best = -1;
        bool best_under = false;
        std::int64_t best_freed = -1, best_peak = 0;
        double best_prog = 2.0;
        int target = -1;
        if (mode == kRounds) {
            while (!left[static_cast<size_t>(turn % G)]) ++turn;
            target = turn++ % G;
        }
        for (int du = 0; du < ndu; ++du) {
            if (done[static_cast<size_t>(du)]) continue;
            const int g = gpu_dst(du / U.nb);
            if (target >= 0 && g != target) continue;
            const std::int64_t during = live[static_cast<size_t>(g)] + w_dst[static_cast<size_t>(du)];
            std::int64_t freed = 0;
            for (int su : reads[static_cast<size_t>(du)])
                if (remaining[static_cast<size_t>(su)] == 1 && gpu_src(su / U.nb) == g) freed += w_src[static_cast<size_t>(su)];
            if (!peak_first) {
                freed = 0;
                for (int su : reads[static_cast<size_t>(du)])
                    if (remaining[static_cast<size_t>(su)] == 1) freed += w_src[static_cast<size_t>(su)];
            }
            const bool under = during <= peak;
            bool take;
            if (best < 0) take = true;
            else if (!peak_first) take = freed > best_freed;
            else if (under != best_under) take = under;
            else if (under && mode == kSpread)
                take = progress(g) < best_prog || (progress(g) == best_prog && freed > best_freed);
            else if (under) take = freed > best_freed;
            else take = during < best_peak || (during == best_peak && freed > best_freed);
            if (take) best = du, best_under = under, best_freed = freed, best_peak = during, best_prog = progress(g);
        }
        done[static_cast<size_t>(best)] = 1;
        order.push_back(best);
        const int g = gpu_dst(best / U.nb);
        --left[static_cast<size_t>(g)];
        live[static_cast<size_t>(g)] += w_dst[static_cast<size_t>(best)];
        peak = std::max(peak, live[static_cast<size_t>(g)]);
        for (int su : reads[static_cast<size_t>(best)])
            if (--remaining[static_cast<size_t>(su)] == 0) live[static_cast<size_t>(gpu_src(su / U.nb))] -= w_src[static_cast<size_t>(su)];
    }
    return {order, peak};
}

}  // namespace

std::vector<int> greedy_stage_order(const core::PlanCore& P, const std::vector<exec::CopyOp>& ops, int bands,
                                    int n_gpus) {
    // both heuristics, keep the lower modeled peak (a global criterion: every rank picks
    // the same order)
    auto a = greedy_pass(P, ops, bands, n_gpus, kFreed);
    auto b = greedy_pass(P, ops, bands, n_gpus, kPeak);
    auto& best = b.second < a.second ? b : a;
    if (n_gpus > 1) {  // across GPUs, spreading wins ties: merged groups keep more links busy
        auto c = greedy_pass(P, ops, bands, n_gpus, kSpread);
        if (c.second <= best.second) return c.first;
    }
    return best.first;
}

namespace {
MemoryPlan plan_with_order(const core::PlanCore& ab, const core::PlanCore* ba, const std::vector<exec::CopyOp>& ops_ab,
                           const std::vector<exec::CopyOp>& ops_ba, std::int64_t C, bool with_grads, int n_gpus, int gpu,
                           int groups, int bands, const std::vector<int>& order_ab);
}  // namespace

MemoryPlan plan_memory(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t C, bool with_grads, int n_gpus,
                       int gpu, int groups, int bands) {
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    const std::vector<exec::CopyOp> ops_ba = ba ? exec::build_ops(*ba) : std::vector<exec::CopyOp>{};
    return plan_memory_ops(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, groups, bands);
}

MemoryPlan plan_memory_ops(const core::PlanCore& ab, const core::PlanCore* ba, const std::vector<exec::CopyOp>& ops_ab,
                           const std::vector<exec::CopyOp>& ops_ba, std::int64_t C, bool with_grads, int n_gpus, int gpu,
                           int groups, int bands) {
    if (groups == kBandInterleaved) {
        // bands in an order that takes one band from each source pipeline stage per
        // group, all destination ranks of a band together: every group draws on every
        // source GPU and feeds every destination GPU, and each group's new data can reuse
        // the old chunks of the groups before it
        const UnitMap U(ab, bands);
        const int S = interleave_stride(ab, U.nb);
        std::vector<int> order;
        for (int i = 0; i < U.nb; ++i) {
            const int band = (i % S) * (U.nb / S) + i / S;
            for (int j = 0; j < U.nd; ++j) order.push_back(j * U.nb + band);
        }
        return plan_with_order(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, U.nb / S, bands, order);
    }
    if (groups < 0) {  // rounds: one unit per GPU per group
        const int G = std::max(1, n_gpus);
        const int units = UnitMap(ab, bands).count();
        return plan_with_order(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, (units + G - 1) / G, bands,
                               greedy_pass(ab, ops_ab, bands, n_gpus, kRounds).first);
    }
    if (n_gpus > 1)  // the order must be global: the modeled-peak choice
        return plan_with_order(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, groups, bands,
                               greedy_stage_order(ab, ops_ab, bands, n_gpus));
    // one GPU: both greedy orders, keep the smaller footprint
    MemoryPlan a = plan_with_order(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, groups, bands,
                                   greedy_pass(ab, ops_ab, bands, n_gpus, kFreed).first);
    MemoryPlan b = plan_with_order(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, groups, bands,
                                   greedy_pass(ab, ops_ab, bands, n_gpus, kPeak).first);
    return b.stats.physical_bytes < a.stats.physical_bytes ? b : a;
}

namespace {
MemoryPlan plan_with_order(const core::PlanCore& ab, const core::PlanCore* ba, const std::vector<exec::CopyOp>& ops_ab,
                           const std::vector<exec::CopyOp>& ops_ba, std::int64_t C, bool with_grads, int n_gpus, int gpu,
                           int groups, int bands, const std::vector<int>& order_ab) {
    MemoryPlan mp;
    mp.chunk = C;
    const UnitMap Uab(ab, bands);
    mp.bands = Uab.nb;
    // contiguous-block placement of the plan's devices (executor.cu gpu_of_phys)
    const int per = gpu_block(ab, n_gpus);
    for (int l = 0; l < 2; ++l) {
        const int nr = l == 0 ? ab.src_cfg.world_size() : ab.dst_cfg.world_size();
        mp.bufs[l].resize(static_cast<size_t>(nr) * exec::kNumBufs);
        for (int r = 0; r < nr; ++r) {
            std::int64_t b[exec::kNumBufs];
            exec::buffer_sizes(ab, l, r, with_grads, b);
            const int phys = l == 0 ? ab.wm.src_phys[static_cast<size_t>(r)] : ab.wm.dst_phys[static_cast<size_t>(r)];
            for (int k = 0; k < exec::kNumBufs; ++k) {
                BufPlan& m = mp.bufs[l][static_cast<size_t>(r) * exec::kNumBufs + k];
                m.bytes = b[k];
                m.remote = phys / per != gpu;  // planned by the GPU that hosts it
                m.direct = m.remote || b[k] < C / 4;  // small buffers (scalars) are plain allocations
                m.reserved = m.direct ? 0 : (b[k] + C - 1) / C * C;
                m.phys.assign(static_cast<size_t>(m.reserved / C), -1);
            }
        }
    }
    // ---- stage units (destination rank x layer band) and their order; concurrency
    // groups: position -> group (MemoryAwareChunk: as many steps per
    // stage as memory allows). Lifetimes are measured in groups, so a chunk is reused
    // only by a LATER group.
    auto group_of = [groups](int s, int n) { return groups <= 0 || groups >= n ? s : s * groups / n; };
    mp.order[0] = order_ab;
    mp.groups = groups;
    const int nu_ab = Uab.count();
    const std::vector<int> pos_ab = positions(mp.order[0], static_cast<size_t>(nu_ab));
    auto chunk_vec = [&](int l, int init) {
        std::vector<std::vector<int>> v(mp.bufs[l].size());
        for (size_t i = 0; i < mp.bufs[l].size(); ++i) v[i].assign(mp.bufs[l][i].phys.size(), init);
        return v;
    };
    auto touch = [&](std::vector<std::vector<int>>& tab, int rank, int buf, Extent e, int stage, bool is_max) {
        auto& v = tab[static_cast<size_t>(rank) * exec::kNumBufs + buf];
        for (std::int64_t c = e.lo / C; c <= (e.hi - 1) / C && c < static_cast<std::int64_t>(v.size()); ++c) {
            int& x = v[static_cast<size_t>(c)];
            x = is_max ? std::max(x, stage) : std::min(x, stage);
        }
    };
    // last read (A) / first write (B) group of every chunk
    std::vector<std::vector<int>> lr_ab = chunk_vec(0, -1), fw_ab = chunk_vec(1, kNever);
    for (const exec::CopyOp& op : ops_ab) {
        const int s = group_of(pos_ab[static_cast<size_t>(Uab.unit(op.dst_rank, op.tensor))], nu_ab);
        touch(lr_ab, op.src_side_rank, op.src_buf, src_extent(op), s, true);
        touch(fw_ab, op.dst_rank, op.dst_buf, dst_extent(op), s, false);
    }
    std::vector<std::vector<int>> lr_ba = chunk_vec(1, -1), fw_ba = chunk_vec(0, kNever);
    if (ba) {
        // B->A writes A units; the A units that die last in A->B are rebuilt first
        const UnitMap Uba(*ba, Uab.nb);
        std::vector<int> death(static_cast<size_t>(Uba.count()), -1);
        for (const exec::CopyOp& op : ops_ab) {
            if (op.tensor < 0) continue;  // the scalar blob is not chunked memory
            const int u = Uba.unit(op.src_side_rank, op.tensor);
            death[static_cast<size_t>(u)] =
                std::max(death[static_cast<size_t>(u)], pos_ab[static_cast<size_t>(Uab.unit(op.dst_rank, op.tensor))]);
        }
        mp.order[1].resize(static_cast<size_t>(Uba.count()));
        for (int u = 0; u < Uba.count(); ++u) mp.order[1][static_cast<size_t>(u)] = u;
        std::sort(mp.order[1].begin(), mp.order[1].end(), [&](int a, int b) {
            const int da = death[static_cast<size_t>(a)], db = death[static_cast<size_t>(b)];
            return da != db ? da > db : a > b;
        });
        const int nu_ba = Uba.count();
        const std::vector<int> pos_ba = positions(mp.order[1], static_cast<size_t>(nu_ba));
        for (const exec::CopyOp& op : ops_ba) {
            const int s = group_of(pos_ba[static_cast<size_t>(Uba.unit(op.dst_rank, op.tensor))], nu_ba);
            touch(lr_ba, op.src_side_rank, op.src_buf, src_extent(op), s, true);
            touch(fw_ba, op.dst_rank, op.dst_buf, dst_extent(op), s, false);
        }
    }
    // ---- assignment: every A chunk owns a physical chunk; a B chunk takes a dead A
    // chunk (LR_AB(a) < FW_AB(b), and LR_BA(b) < FW_BA(a) for round trips; tightest
    // FW_BA first) or a fresh one
    struct AChunk {
        int lr_ab, fw_ba, phys;
    };
    std::vector<AChunk> achunks;
    int nphys = 0;
    for (size_t i = 0; i < mp.bufs[0].size(); ++i) {
        BufPlan& m = mp.bufs[0][i];
        for (size_t c = 0; c < m.phys.size(); ++c) {
            m.phys[c] = nphys++;
            achunks.push_back({lr_ab[i][c], fw_ba[i][c], m.phys[c]});
        }
    }
    mp.stats.a_bytes = static_cast<std::int64_t>(nphys) * C;
    struct BChunk {
        int fw_ab, lr_ba;
        size_t buf, idx;
    };
    std::vector<BChunk> bchunks;
    for (size_t i = 0; i < mp.bufs[1].size(); ++i)
        for (size_t c = 0; c < mp.bufs[1][i].phys.size(); ++c) bchunks.push_back({fw_ab[i][c], lr_ba[i][c], i, c});
    std::stable_sort(bchunks.begin(), bchunks.end(), [](const BChunk& a, const BChunk& b) { return a.fw_ab < b.fw_ab; });
    std::vector<size_t> aorder(achunks.size());
    for (size_t i = 0; i < aorder.size(); ++i) aorder[i] = i;
    std::stable_sort(aorder.begin(), aorder.end(), [&](size_t a, size_t b) { return achunks[a].lr_ab < achunks[b].lr_ab; });
    std::multimap<int, int> avail;  // FW_BA(a) -> physical chunk
    size_t ai = 0;
    int fresh = 0;
    for (const BChunk& b : bchunks) {
        while (ai < aorder.size() && achunks[aorder[ai]].lr_ab < b.fw_ab) {
            const AChunk& a = achunks[aorder[ai++]];
            avail.emplace(ba ? a.fw_ba : 0, a.phys);
        }
        int p = -1;
        if (!avail.empty()) {
            auto it = ba ? avail.upper_bound(b.lr_ba) : avail.begin();
            if (it != avail.end()) {
                p = it->second;
                avail.erase(it);
                mp.stats.aliased_bytes += C;
            }
        }
        if (p < 0) p = nphys + fresh++;
        mp.bufs[1][b.buf].phys[b.idx] = p;
    }
    mp.nphys = nphys + fresh;
    mp.stats.chunks = mp.nphys;
    mp.stats.physical_bytes = static_cast<std::int64_t>(mp.nphys) * C;
    for (const BufPlan& m : mp.bufs[1])
        if (!m.remote) mp.stats.b_bytes += m.bytes;
    plan_stage_cuts(mp, ab, ba, ops_ab, ops_ba);
    return mp;
}
}  // namespace

std::vector<ScheduleLevel> schedule_levels(const core::PlanCore& ab, int n_gpus) {
    std::vector<ScheduleLevel> v;
    const int nd = ab.dst_cfg.world_size();
    const int L = std::max(1, ab.space->num_layers());
    const int G = std::max(1, n_gpus);
    for (int nb = 1;; nb *= 2) {
        const int n = std::min(nb, L);
        const int units = nd * n;
        const int rounds = (units + G - 1) / G;
        // group counts 1, 2, 4, ... and finally one group per unit: each count refines the
        // previous one (nested boundaries), so within a band count more groups never alias
        // less. Across GPUs the rounds order (one unit per GPU per group, groups = -1) comes
        // before the levels with as many or more groups: same barriers, every link busy.
        std::vector<int> ks;
        for (int k = 1; k < units; k *= 2) ks.push_back(k);
        ks.push_back(units);
        bool rounds_done = G < 2 || rounds < 2;
        // across GPUs: the band-interleaved order (every group spans every GPU's links)
        if (G >= 2 && n >= 2) v.push_back({n, kBandInterleaved});
        for (int k : ks) {
            if (!rounds_done && k >= rounds) {
                v.push_back({n, -1});
                rounds_done = true;
            }
            if (!(n > 1 && k == 1)) v.push_back({n, k});  // one group is the same at any band count
        }
        if (n >= L) break;
    }
    return v;
}

int choose_schedule(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t C, bool with_grads, int n_gpus,
                    int gpu, std::int64_t cap, std::int64_t* physical) {
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    const std::vector<exec::CopyOp> ops_ba = ba ? exec::build_ops(*ba) : std::vector<exec::CopyOp>{};
    const std::vector<ScheduleLevel> levels = schedule_levels(ab, n_gpus);
    std::int64_t best = std::numeric_limits<std::int64_t>::max();
    for (size_t i = 0; i < levels.size();) {
        // a band count whose most-aliased plan does not fit is skipped whole: its other
        // levels alias less
        size_t last = i;
        while (last + 1 < levels.size() && levels[last + 1].bands == levels[i].bands) ++last;
        const MemoryPlan most =
            plan_memory_ops(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, levels[last].groups, levels[last].bands);
        best = std::min(best, most.stats.physical_bytes);
        if (most.stats.physical_bytes <= cap)
            for (size_t j = i; j <= last; ++j) {
                const std::int64_t phys =
                    j == last ? most.stats.physical_bytes
                              : plan_memory_ops(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, levels[j].groups,
                                                levels[j].bands)
                                    .stats.physical_bytes;
                if (phys <= cap) {
                    if (physical) *physical = phys;
                    return static_cast<int>(j);
                }
            }
        i = last + 1;
    }
    if (physical) *physical = best;
    return -1;
}

std::vector<std::int64_t> schedule_footprints(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t C,
                                              bool with_grads, int n_gpus, int gpu) {
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    const std::vector<exec::CopyOp> ops_ba = ba ? exec::build_ops(*ba) : std::vector<exec::CopyOp>{};
    std::vector<std::int64_t> out;
    for (const ScheduleLevel& L : schedule_levels(ab, n_gpus))
        out.push_back(plan_memory_ops(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, L.groups, L.bands).stats.physical_bytes);
    return out;
}

double estimate_seconds(const MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba,
                        const std::vector<exec::CopyOp>& ops_ab, const std::vector<exec::CopyOp>& ops_ba, int n_gpus) {
    // a stage group runs as one launch per GPU: its time is the busiest GPU's bound —
    // NVLink out, NVLink in, or HBM (local copies read + write, peer traffic once) — plus
    // one barrier; groups run one after another
    constexpr double kNvlink = 690e9, kHbm = 6200e9, kBarrier = 30e-6;
    const int G = std::max(1, n_gpus);
    double total = 0.0;
    for (int d = 0; d < (ba ? 2 : 1); ++d) {
        const core::PlanCore& P = d == 0 ? ab : *ba;
        const std::vector<exec::CopyOp>& ops = d == 0 ? ops_ab : ops_ba;
        const UnitMap U(P, mp.bands);
        const std::vector<int> pos = positions(mp.order[d], static_cast<size_t>(U.count()));
        std::vector<int> grp(mp.order[d].size(), 0);
        int ng = 0;
        for (size_t s = 0; s < grp.size(); ++s) {
            if (s == 0 || (s < mp.cut[d].size() && mp.cut[d][s])) ++ng;
            grp[s] = ng - 1;
        }
        ng = std::max(ng, 1);
        const int per = gpu_block(P, G);
        std::vector<double> out(static_cast<size_t>(ng) * G, 0.0), in(out.size(), 0.0), loc(out.size(), 0.0);
        for (const exec::CopyOp& op : ops) {
            const int gs = P.wm.src_phys[static_cast<size_t>(op.src_side_rank)] / per;
            const int gd = P.wm.dst_phys[static_cast<size_t>(op.dst_rank)] / per;
            const size_t k = static_cast<size_t>(grp[static_cast<size_t>(pos[static_cast<size_t>(U.unit(op.dst_rank, op.tensor))])]);
            const double b = static_cast<double>(op.rows) * static_cast<double>(op.row_bytes);
            if (gs == gd) loc[k * G + gs] += b;
            else out[k * G + gs] += b, in[k * G + gd] += b;
        }
        for (int k = 0; k < ng; ++k) {
            double t = 0.0;
            for (int g = 0; g < G; ++g) {
                const size_t i = static_cast<size_t>(k) * G + g;
                t = std::max({t, out[i] / kNvlink, in[i] / kNvlink, (2 * loc[i] + out[i] + in[i]) / kHbm});
            }
            total += t + kBarrier;
        }
    }
    return total;
}

std::vector<std::pair<std::int64_t, double>> schedule_costs(const core::PlanCore& ab, const core::PlanCore* ba,
                                                            std::int64_t C, bool with_grads, int n_gpus, int gpu) {
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    const std::vector<exec::CopyOp> ops_ba = ba ? exec::build_ops(*ba) : std::vector<exec::CopyOp>{};
    std::vector<std::pair<std::int64_t, double>> out;
    const int G = std::max(1, n_gpus);
    const pool::Warm warm;
    for (const ScheduleLevel& L : schedule_levels(ab, n_gpus)) {
        // the run barriers wherever ANY GPU's aliasing needs a cut (runtime.global_stage_cuts),
        // so the level is modeled with the union of every GPU's cuts (each GPU plans only
        // the chunks it hosts; the stage order is common)
        std::vector<MemoryPlan> mps(static_cast<size_t>(G));
        pool::parallel_for(mps.size(), [&](size_t g) {
            mps[g] = plan_memory_ops(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, static_cast<int>(g), L.groups, L.bands);
        });
        MemoryPlan& mp = mps[static_cast<size_t>(gpu)];
        const std::int64_t physical = mp.stats.physical_bytes;
        for (int d = 0; d < 2; ++d)
            for (const MemoryPlan& o : mps) {
                if (o.cut[d].size() > mp.cut[d].size()) mp.cut[d].resize(o.cut[d].size(), 0);
                for (size_t s = 0; s < o.cut[d].size(); ++s) mp.cut[d][s] = mp.cut[d][s] || o.cut[d][s];
            }
        out.push_back({physical, estimate_seconds(mp, ab, ba, ops_ab, ops_ba, n_gpus)});
    }
    return out;
}

int min_stage_groups(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t C, bool with_grads, int n_gpus,
                     int gpu, std::int64_t cap, std::int64_t* physical) {
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    const std::vector<exec::CopyOp> ops_ba = ba ? exec::build_ops(*ba) : std::vector<exec::CopyOp>{};
    const int n = std::max(ab.dst_cfg.world_size(), ba ? ba->dst_cfg.world_size() : 0);
    for (int k = 1; k <= n; ++k) {
        const MemoryPlan mp = plan_memory_ops(ab, ba, ops_ab, ops_ba, C, with_grads, n_gpus, gpu, k, 1);
        if (physical) *physical = mp.stats.physical_bytes;
        if (mp.stats.physical_bytes <= cap) return k;
    }
    return -1;
}

namespace {

// per stage position of one direction: physical chunks read, and (chunk, new owner) written
struct StageIo {
    std::vector<int> reads;  // (chunk, expected owner buffer, expected owner chunk) triples
    std::vector<std::pair<int, Owner>> writes;
};

std::vector<StageIo> stage_io(const MemoryPlan& mp, const core::PlanCore& P, const std::vector<exec::CopyOp>& ops,
                              const std::vector<int>& order, int src_layout) {
    const std::int64_t C = mp.chunk;
    const UnitMap U(P, mp.bands);
    const std::vector<int> pos = positions(order, static_cast<size_t>(U.count()));
    const int dst_layout = 1 - src_layout;
    std::vector<StageIo> io(order.size());
    for (const exec::CopyOp& op : ops) {
        StageIo& st = io[static_cast<size_t>(pos[static_cast<size_t>(U.unit(op.dst_rank, op.tensor))])];
        const size_t sb = static_cast<size_t>(op.src_side_rank) * exec::kNumBufs + op.src_buf;
        const size_t db = static_cast<size_t>(op.dst_rank) * exec::kNumBufs + op.dst_buf;
        const BufPlan& S = mp.bufs[src_layout][sb];
        const BufPlan& D = mp.bufs[dst_layout][db];
        if (!S.direct) {
            const Extent e = src_extent(op);
            for (std::int64_t c = e.lo / C; c <= (e.hi - 1) / C; ++c) {
                st.reads.push_back(S.phys[static_cast<size_t>(c)]);
                st.reads.push_back(static_cast<int>(sb));
                st.reads.push_back(static_cast<int>(c));
            }
        }
        if (!D.direct) {
            const Extent e = dst_extent(op);
            for (std::int64_t c = e.lo / C; c <= (e.hi - 1) / C; ++c)
                st.writes.push_back({D.phys[static_cast<size_t>(c)], Owner{dst_layout, db, static_cast<size_t>(c)}});
        }
    }
    return io;
}

}  // namespace

void plan_stage_cuts(MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba,
                     const std::vector<exec::CopyOp>& ops_ab, const std::vector<exec::CopyOp>& ops_ba) {
    // greedy maximal groups of consecutive stages: a stage joins the running group unless
    // it writes a physical chunk that an earlier stage of the group reads (the aliased
    // old data would be clobbered while still being copied)
    for (int d = 0; d < (ba ? 2 : 1); ++d) {
        const std::vector<StageIo> io = stage_io(mp, d == 0 ? ab : *ba, d == 0 ? ops_ab : ops_ba, mp.order[d], d);
        mp.cut[d].assign(io.size(), 0);
        std::vector<char> read_in_group(static_cast<size_t>(mp.nphys), 0);
        std::vector<int> touched;
        auto add_reads = [&](size_t s) {
            for (size_t k = 0; k < io[s].reads.size(); k += 3) {
                const int p = io[s].reads[k];
                if (!read_in_group[static_cast<size_t>(p)]) read_in_group[static_cast<size_t>(p)] = 1, touched.push_back(p);
            }
        };
        // aliasing only crosses the plan's concurrency groups, so a needed cut may move back
        // to the start of its group: every GPU then cuts on the same group boundaries and
        // the union over GPUs (runtime.global_stage_cuts) stays at most one cut per group
        const int n = static_cast<int>(io.size());
        auto group = [&](int x) { return mp.groups <= 0 || mp.groups >= n ? x : x * mp.groups / n; };
        int last_cut = 0;
        for (size_t s = 0; s < io.size(); ++s) {
            bool conflict = false;
            for (const auto& w : io[s].writes) conflict = conflict || read_in_group[static_cast<size_t>(w.first)];
            if (conflict) {
                int b = static_cast<int>(s);
                while (b - 1 > last_cut && group(b - 1) == group(static_cast<int>(s))) --b;
                mp.cut[d][static_cast<size_t>(b)] = 1;
                last_cut = b;
                for (int p : touched) read_in_group[static_cast<size_t>(p)] = 0;
                touched.clear();
                for (int q = b; q < static_cast<int>(s); ++q) add_reads(static_cast<size_t>(q));
                // the moved cut relies on aliasing never occurring inside a concurrency
                // group: stage s must not write what the rebuilt group (b..s-1) reads
                for (const auto& w : io[s].writes)
                    if (read_in_group[static_cast<size_t>(w.first)])
                        throw std::logic_error(strfmt("memory plan: stage %zu writes chunk %d that stage group "
                                                      "starting at %d still reads (aliasing inside a group)",
                                                      s, w.first, b));
            }
            add_reads(s);
        }
        if (!mp.cut[d].empty()) mp.cut[d][0] = 1;
    }
}

std::vector<std::vector<int>> last_read_stage(const MemoryPlan& mp, const core::PlanCore& ab,
                                              const std::vector<exec::CopyOp>& ops_ab) {
    // executed stage of each position: positions between two cuts share one launch group
    const std::vector<StageIo> io = stage_io(mp, ab, ops_ab, mp.order[0], 0);
    std::vector<int> stage(io.size(), 0);
    int st = -1;
    for (size_t s = 0; s < io.size(); ++s) {
        if (s == 0 || (s < mp.cut[0].size() && mp.cut[0][s])) ++st;
        stage[s] = st;
    }
    std::vector<std::vector<int>> out(mp.bufs[0].size());
    for (size_t i = 0; i < mp.bufs[0].size(); ++i) out[i].assign(mp.bufs[0][i].phys.size(), -1);
    for (size_t s = 0; s < io.size(); ++s)
        for (size_t k = 0; k < io[s].reads.size(); k += 3) {
            int& x = out[static_cast<size_t>(io[s].reads[k + 1])][static_cast<size_t>(io[s].reads[k + 2])];
            x = std::max(x, stage[s]);
        }
    return out;
}

std::int64_t simulate_memory_plan(const MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba) {
    // owner[p] = (layout, buffer index, chunk index) whose data physical chunk p holds;
    // stages between two cuts run concurrently (one group), groups run in order
    std::vector<Owner> owner(static_cast<size_t>(mp.nphys));
    for (size_t i = 0; i < mp.bufs[0].size(); ++i)
        for (size_t c = 0; c < mp.bufs[0][i].phys.size(); ++c) owner[static_cast<size_t>(mp.bufs[0][i].phys[c])] = {0, i, c};
    std::int64_t violations = 0;
    for (int d = 0; d < (ba ? 2 : 1); ++d) {
        const core::PlanCore& P = d == 0 ? ab : *ba;
        const std::vector<StageIo> io = stage_io(mp, P, exec::build_ops(P), mp.order[d], d);
        const int src_layout = d;
        size_t s = 0;
        while (s < io.size()) {
            size_t e = s + 1;
            while (e < io.size() && !(e < mp.cut[d].size() && mp.cut[d][e])) ++e;
            std::vector<char> read_now(static_cast<size_t>(mp.nphys), 0);
            for (size_t t = s; t < e; ++t)
                for (size_t k = 0; k < io[t].reads.size(); k += 3) {
                    const int p = io[t].reads[k];
                    const Owner& o = owner[static_cast<size_t>(p)];
                    if (o.layout != src_layout || o.buf != static_cast<size_t>(io[t].reads[k + 1]) ||
                        o.chunk != static_cast<size_t>(io[t].reads[k + 2]))
                        ++violations;
                    read_now[static_cast<size_t>(p)] = 1;
                }
            for (size_t t = s; t < e; ++t)
                for (const auto& w : io[t].writes) {
                    const Owner& o = owner[static_cast<size_t>(w.first)];
                    if (read_now[static_cast<size_t>(w.first)] && !(o.layout == w.second.layout && o.buf == w.second.buf))
                        ++violations;
                }
            for (size_t t = s; t < e; ++t)
                for (const auto& w : io[t].writes) owner[static_cast<size_t>(w.first)] = w.second;
            s = e;
        }
    }
    return violations;
}

}  // namespace mem
}  // namespace reshard
