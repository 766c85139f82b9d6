// Host side of the memory-aware arena (arena.hpp): stage orders, chunk lifetimes,
// the aliasing assignment, and an independent execution simulation that checks it.
#include <algorithm>
#include <limits>
#include <map>

#include "reshard/arena.hpp"

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

}  // namespace

std::vector<int> greedy_stage_order(const core::PlanCore& P, const std::vector<exec::CopyOp>& ops) {
    const int ns = P.src_cfg.world_size(), nd = P.dst_cfg.world_size();
    std::vector<std::vector<char>> reads(static_cast<size_t>(ns), std::vector<char>(static_cast<size_t>(nd), 0));
    for (const exec::CopyOp& op : ops) reads[static_cast<size_t>(op.src_side_rank)][static_cast<size_t>(op.dst_rank)] = 1;
    std::vector<std::int64_t> sbytes(static_cast<size_t>(ns), 0);
    for (int i = 0; i < ns; ++i) {
        std::int64_t b[exec::kNumBufs];
        exec::buffer_sizes(P, 0, i, false, b);
        for (int k = 0; k < exec::kNumBufs; ++k) sbytes[static_cast<size_t>(i)] += b[k];
    }
    std::vector<char> done(static_cast<size_t>(nd), 0), dead(static_cast<size_t>(ns), 0);
    auto all_consumers_done = [&](int i, int extra) {
        for (int d = 0; d < nd; ++d)
            if (reads[static_cast<size_t>(i)][static_cast<size_t>(d)] && !done[static_cast<size_t>(d)] && d != extra) return false;
        return true;
    };
    std::vector<int> order;
    for (int step = 0; step < nd; ++step) {
        int best = -1;
        std::int64_t best_freed = -1;
        for (int j = 0; j < nd; ++j) {
            if (done[static_cast<size_t>(j)]) continue;
            std::int64_t freed = 0;
            for (int i = 0; i < ns; ++i)
                if (!dead[static_cast<size_t>(i)] && all_consumers_done(i, j)) freed += sbytes[static_cast<size_t>(i)];
            if (freed > best_freed) best = j, best_freed = freed;
        }
        done[static_cast<size_t>(best)] = 1;
        order.push_back(best);
        for (int i = 0; i < ns; ++i)
            if (all_consumers_done(i, -1)) dead[static_cast<size_t>(i)] = 1;
    }
    return order;
}

MemoryPlan plan_memory(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t C, bool with_grads, int n_gpus,
                       int gpu, int groups) {
    MemoryPlan mp;
    mp.chunk = C;
    // stage position -> concurrency group (MemoryAwareChunk: as many
    // steps per stage as memory allows); lifetimes are measured in groups, so a chunk is
    // reused only by a LATER group
    auto group_of = [groups](int s, int n) { return groups <= 0 || groups >= n ? s : s * groups / n; };
    // contiguous-block placement of the plan's devices (executor.cu gpu_of_phys)
    int max_phys = 0;
    for (const auto& r : ab.routes) max_phys = std::max(max_phys, r.phys);
    const int per = (max_phys + 1 + n_gpus - 1) / n_gpus;
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
    // ---- lifetimes: last read (A) / first write (B) stage of every chunk
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    mp.order[0] = greedy_stage_order(ab, ops_ab);
    const std::vector<int> pos_ab = positions(mp.order[0], static_cast<size_t>(ab.dst_cfg.world_size()));
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
    std::vector<std::vector<int>> lr_ab = chunk_vec(0, -1), fw_ab = chunk_vec(1, kNever);
    for (const exec::CopyOp& op : ops_ab) {
        const int s = group_of(pos_ab[static_cast<size_t>(op.dst_rank)], ab.dst_cfg.world_size());
        touch(lr_ab, op.src_side_rank, op.src_buf, src_extent(op), s, true);
        touch(fw_ab, op.dst_rank, op.dst_buf, dst_extent(op), s, false);
    }
    std::vector<std::vector<int>> lr_ba = chunk_vec(1, -1), fw_ba = chunk_vec(0, kNever);
    if (ba) {
        // B->A writes A ranks; A ranks that die last in A->B are rebuilt first
        const int na = ab.src_cfg.world_size();
        std::vector<int> death(static_cast<size_t>(na), -1);
        for (int r = 0; r < na; ++r)
            for (int k = 0; k < exec::kNumBufs; ++k)
                for (int x : lr_ab[static_cast<size_t>(r) * exec::kNumBufs + k])
                    death[static_cast<size_t>(r)] = std::max(death[static_cast<size_t>(r)], x);
        mp.order[1].resize(static_cast<size_t>(na));
        for (int r = 0; r < na; ++r) mp.order[1][static_cast<size_t>(r)] = r;
        std::sort(mp.order[1].begin(), mp.order[1].end(), [&](int a, int b) {
            const int da = death[static_cast<size_t>(a)], db = death[static_cast<size_t>(b)];
            return da != db ? da > db : a > b;
        });
        const std::vector<int> pos_ba = positions(mp.order[1], static_cast<size_t>(na));
        for (const exec::CopyOp& op : exec::build_ops(*ba)) {
            const int s = group_of(pos_ba[static_cast<size_t>(op.dst_rank)], na);
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
    plan_stage_cuts(mp, ab, ba);
    return mp;
}

namespace {

// per stage position of one direction: physical chunks read, and (chunk, new owner) written
struct StageIo {
    std::vector<int> reads;
    std::vector<std::pair<int, Owner>> writes;
};

std::vector<StageIo> stage_io(const MemoryPlan& mp, const core::PlanCore& P, const std::vector<int>& order, int src_layout) {
    const std::int64_t C = mp.chunk;
    const std::vector<exec::CopyOp> ops = exec::build_ops(P);
    const std::vector<int> pos = positions(order, static_cast<size_t>(P.dst_cfg.world_size()));
    const int dst_layout = 1 - src_layout;
    std::vector<StageIo> io(order.size());
    for (const exec::CopyOp& op : ops) {
        StageIo& st = io[static_cast<size_t>(pos[static_cast<size_t>(op.dst_rank)])];
        const size_t sb = static_cast<size_t>(op.src_side_rank) * exec::kNumBufs + op.src_buf;
        const size_t db = static_cast<size_t>(op.dst_rank) * exec::kNumBufs + op.dst_buf;
        const BufPlan& S = mp.bufs[src_layout][sb];
        const BufPlan& D = mp.bufs[dst_layout][db];
        if (!S.direct) {
            const Extent e = src_extent(op);
            for (std::int64_t c = e.lo / C; c <= (e.hi - 1) / C; ++c) {
                st.reads.push_back(S.phys[static_cast<size_t>(c)]);
                st.reads.push_back(static_cast<int>(sb));  // (chunk, expected owner) pairs
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

void plan_stage_cuts(MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba) {
    // greedy maximal groups of consecutive stages: a stage joins the running group unless
    // it writes a physical chunk that an earlier stage of the group reads (the aliased
    // old data would be clobbered while still being copied)
    for (int d = 0; d < (ba ? 2 : 1); ++d) {
        const std::vector<StageIo> io = stage_io(mp, d == 0 ? ab : *ba, mp.order[d], d);
        mp.cut[d].assign(io.size(), 0);
        std::vector<char> read_in_group(static_cast<size_t>(mp.nphys), 0);
        std::vector<int> touched;
        for (size_t s = 0; s < io.size(); ++s) {
            bool conflict = false;
            for (const auto& w : io[s].writes) conflict = conflict || read_in_group[static_cast<size_t>(w.first)];
            if (conflict) {
                mp.cut[d][s] = 1;
                for (int p : touched) read_in_group[static_cast<size_t>(p)] = 0;
                touched.clear();
            }
            for (size_t k = 0; k < io[s].reads.size(); k += 3) {
                const int p = io[s].reads[k];
                if (!read_in_group[static_cast<size_t>(p)]) read_in_group[static_cast<size_t>(p)] = 1, touched.push_back(p);
            }
        }
        if (!mp.cut[d].empty()) mp.cut[d][0] = 1;
    }
}

int min_stage_groups(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t C, bool with_grads, int n_gpus,
                     int gpu, std::int64_t cap, std::int64_t* physical) {
    const int n = std::max(ab.dst_cfg.world_size(), ba ? ba->dst_cfg.world_size() : 0);
    for (int k = 1; k <= n; ++k) {
        const MemoryPlan mp = plan_memory(ab, ba, C, with_grads, n_gpus, gpu, k);
        if (physical) *physical = mp.stats.physical_bytes;
        if (mp.stats.physical_bytes <= cap) return k;
    }
    return -1;
}

std::int64_t simulate_memory_plan(const MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba) {
    // owner[p] = (layout, buffer index, chunk index) whose data physical chunk p holds;
    // stages between two cuts run concurrently (one group), groups run in order
    std::vector<Owner> owner(static_cast<size_t>(mp.nphys));
    for (size_t i = 0; i < mp.bufs[0].size(); ++i)
        for (size_t c = 0; c < mp.bufs[0][i].phys.size(); ++c) owner[static_cast<size_t>(mp.bufs[0][i].phys[c])] = {0, i, c};
    std::int64_t violations = 0;
    for (int d = 0; d < (ba ? 2 : 1); ++d) {
        const std::vector<StageIo> io = stage_io(mp, d == 0 ? ab : *ba, mp.order[d], d);
        const int src_layout = d;
        size_t s = 0;
        while (s < io.size()) {
            size_t e = s + 1;
            while (e < io.size() && !(d < 2 && e < mp.cut[d].size() && mp.cut[d][e])) ++e;
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
