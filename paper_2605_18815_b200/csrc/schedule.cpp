// Algorithm 1 transition schedule (schedule.hpp).
#include "reshard/schedule.hpp"

#include <algorithm>
#include <map>
#include <numeric>

#include "reshard/executor_rt.hpp"

namespace reshard {
namespace sched {

std::vector<int> xor_steps(int N) {
    int p = 1;
    while (p < N) p <<= 1;
    std::vector<int> s;
    for (int i = 1; i < p; ++i) s.push_back(i);
    return s;
}

std::vector<std::vector<int>> memory_aware_chunk(const std::vector<int>& steps, const std::vector<std::int64_t>& cost,
                                                 const std::vector<std::int64_t>& mem_avail, std::int64_t* budget) {
    if (mem_avail.empty()) throw ConfigError("memory_aware_chunk needs at least one rank budget");
    // AllReduce(M_avail, MIN): every rank computes the same global minimum
    const std::int64_t M = *std::min_element(mem_avail.begin(), mem_avail.end());
    if (budget) *budget = M;
    std::vector<std::vector<int>> stages;
    std::vector<int> cur;
    std::int64_t used = 0;
    for (int s : steps) {
        const std::int64_t c = cost[static_cast<size_t>(s)];
        if (c > M)
            throw exec::BudgetError(strfmt("infeasible budget: finer fragmentation required (step %d needs %lld bytes, "
                                           "budget %lld)", s, static_cast<long long>(c), static_cast<long long>(M)));
        if (used + c > M && !cur.empty()) {
            stages.push_back(cur);
            cur.assign(1, s);
            used = c;
        } else {
            cur.push_back(s);
            used += c;
        }
    }
    if (!cur.empty()) stages.push_back(cur);
    return stages;
}

std::vector<Fragment> plan_fragments(const core::PlanCore& P, const std::vector<core::FlatXfer>& flat) {
    std::map<int, int> dev_of_phys;
    for (size_t i = 0; i < P.routes.size(); ++i) dev_of_phys[P.routes[i].phys] = static_cast<int>(i);
    std::vector<Fragment> out;
    out.reserve(P.box.size() + flat.size());
    size_t bi = 0, fi = 0;
    while (bi < P.box.size() || fi < flat.size()) {
        bool take_box;
        if (bi == P.box.size()) take_box = false;
        else if (fi == flat.size()) take_box = true;
        else {
            const auto& b = P.box[bi];
            const auto& f = flat[fi];
            take_box = b.src != f.src ? b.src < f.src : b.dst != f.dst ? b.dst < f.dst : b.kind < 1;
        }
        Fragment g;
        if (take_box) {
            const auto& b = P.box[bi++];
            g.kind = b.kind;
            g.tensor = b.tensor;
            for (int d = 0; d < 4; ++d) g.lo[d] = b.lo[d], g.hi[d] = b.hi[d];
            g.src_rank = b.src;
            g.dst_rank = b.dst;
            g.bytes = b.bytes;
        } else {
            const auto& f = flat[fi++];
            g.kind = 1;
            g.lo[0] = f.lo;
            g.hi[0] = f.hi;
            g.src_rank = f.src;
            g.dst_rank = f.dst;
            g.bytes = (f.hi - f.lo) * kOptimStateBytes;
        }
        g.src_dev = dev_of_phys.at(P.wm.src_phys[static_cast<size_t>(g.src_rank)]);
        g.dst_dev = dev_of_phys.at(P.wm.dst_phys[static_cast<size_t>(g.dst_rank)]);
        out.push_back(g);
    }
    return out;
}

namespace {

int frag_nd(const core::PlanCore& P, const Fragment& f) {
    return f.tensor < 0 ? 1 : static_cast<int>(P.space->entries()[static_cast<size_t>(f.tensor)].spec.shape.size());
}

bool same_region(const core::PlanCore& P, const Fragment& a, const Fragment& b) {
    const int nd = frag_nd(P, a);
    for (int d = 0; d < nd; ++d)
        if (a.lo[d] != b.lo[d] || a.hi[d] != b.hi[d]) return false;
    return true;
}

/// IsContiguous: the slices tile one interval along a single axis with no gap.
bool contiguous(const core::PlanCore& P, std::vector<const Fragment*> v) {
    if (v.size() < 2) return true;
    const int nd = frag_nd(P, *v[0]);
    std::sort(v.begin(), v.end(), [nd](const Fragment* a, const Fragment* b) {
        for (int d = 0; d < nd; ++d) {
            if (a->lo[d] != b->lo[d]) return a->lo[d] < b->lo[d];
            if (a->hi[d] != b->hi[d]) return a->hi[d] < b->hi[d];
        }
        return false;
    });
    int axis = -1;
    for (size_t i = 1; i < v.size(); ++i) {
        int diff = -1;
        for (int d = 0; d < nd; ++d) {
            if (v[i]->lo[d] == v[0]->lo[d] && v[i]->hi[d] == v[0]->hi[d]) continue;
            if (diff >= 0) return false;
            diff = d;
        }
        if (diff < 0) return false;  // duplicate slice
        if (axis >= 0 && diff != axis) return false;
        axis = diff;
        if (v[i - 1]->hi[axis] != v[i]->lo[axis]) return false;
    }
    return true;
}

}  // namespace

std::vector<CommOp> optimize_primitives(const core::PlanCore& P, const std::vector<Fragment>& frags,
                                        std::vector<std::int64_t>* residual, bool promote) {
    // GroupByLogicalTensor: (kind, tensor id); flat optimizer runs form one group
    std::map<std::pair<int, int>, std::vector<std::int64_t>> groups;
    for (size_t i = 0; i < frags.size(); ++i) groups[{frags[i].kind, frags[i].tensor}].push_back(static_cast<std::int64_t>(i));
    std::vector<CommOp> out;
    std::vector<char> promoted(frags.size(), 0);
    if (promote) {
        for (auto& [key, idx] : groups) {
            std::vector<int> srcs, dsts;
            std::vector<const Fragment*> fv;
            for (std::int64_t i : idx) {
                fv.push_back(&frags[static_cast<size_t>(i)]);
                srcs.push_back(frags[static_cast<size_t>(i)].src_dev);
                dsts.push_back(frags[static_cast<size_t>(i)].dst_dev);
            }
            for (std::vector<int>* s : {&srcs, &dsts}) {
                std::sort(s->begin(), s->end());
                s->erase(std::unique(s->begin(), s->end()), s->end());
            }
            CommOp op;
            bool identical = true;
            for (const Fragment* f : fv) identical &= same_region(P, *f, *fv[0]);
            // one destination may appear only once for a broadcast / scatter slice set
            const bool one_per_dst = dsts.size() == fv.size();
            if (srcs.size() == 1 && dsts.size() > 1 && one_per_dst && identical) {
                op.kind = CommKind::Broadcast;
                op.root = srcs[0];
            } else if (srcs.size() == 1 && dsts.size() > 1 && one_per_dst && contiguous(P, fv)) {
                op.kind = CommKind::Scatter;
                op.root = srcs[0];
            } else if (srcs.size() > 1 && dsts.size() == 1 && srcs.size() == fv.size() && contiguous(P, fv)) {
                op.kind = CommKind::Gather;
                op.root = dsts[0];
            } else {
                continue;
            }
            op.participants = srcs;
            op.participants.insert(op.participants.end(), dsts.begin(), dsts.end());
            std::sort(op.participants.begin(), op.participants.end());
            op.participants.erase(std::unique(op.participants.begin(), op.participants.end()), op.participants.end());
            op.frags = idx;
            for (std::int64_t i : idx) {
                op.bytes += frags[static_cast<size_t>(i)].bytes;
                promoted[static_cast<size_t>(i)] = 1;
            }
            out.push_back(std::move(op));
        }
    }
    if (residual) {
        residual->clear();
        for (size_t i = 0; i < frags.size(); ++i)
            if (!promoted[i]) residual->push_back(static_cast<std::int64_t>(i));
    }
    return out;
}

TransitionSchedule build_schedule(const core::PlanCore& P, const std::vector<core::FlatXfer>& flat,
                                  const std::vector<std::int64_t>& mem_avail, bool promote) {
    TransitionSchedule T;
    T.N = static_cast<int>(P.routes.size());
    for (const auto& r : P.routes) T.devices.push_back(r.phys);
    T.frags = plan_fragments(P, flat);
    std::vector<std::int64_t> residual;
    T.collectives = optimize_primitives(P, T.frags, &residual, promote);
    // FreeObsoleteBuffers: gradients in drop mode; state of departing devices after send
    T.free_list.resize(static_cast<size_t>(T.N));
    for (int i = 0; i < T.N; ++i) {
        const auto& r = P.routes[static_cast<size_t>(i)];
        if (r.src_rank >= 0 && P.opts.gradients == GradientPolicy::Drop)
            T.free_list[static_cast<size_t>(i)].push_back(strfmt("grad src rank %d", r.src_rank));
        if (r.src_rank >= 0 && r.dst_rank < 0)
            T.free_list[static_cast<size_t>(i)].push_back(strfmt("departing src rank %d (after its sends)", r.src_rank));
    }
    // per (i, j) residual traffic in plan order
    const int N = T.N;
    std::vector<std::vector<std::vector<std::int64_t>>> pair(static_cast<size_t>(N),
                                                               std::vector<std::vector<std::int64_t>>(static_cast<size_t>(N)));
    for (std::int64_t f : residual) {
        const Fragment& g = T.frags[static_cast<size_t>(f)];
        pair[static_cast<size_t>(g.src_dev)][static_cast<size_t>(g.dst_dev)].push_back(f);
    }
    auto bytes_of = [&](int i, int j) {
        std::int64_t b = 0;
        for (std::int64_t f : pair[static_cast<size_t>(i)][static_cast<size_t>(j)]) b += T.frags[static_cast<size_t>(f)].bytes;
        return b;
    };
    const std::vector<int> all_steps = xor_steps(N);
    T.step_cost.assign(all_steps.size() + 1, 0);
    std::vector<int> steps;
    for (int s : all_steps) {
        std::int64_t worst = 0;
        for (int i = 0; i < N; ++i) {
            const int p = xor_peer(i, s, N);
            if (p < 0) continue;
            worst = std::max(worst, bytes_of(i, p) + bytes_of(p, i));
        }
        T.step_cost[static_cast<size_t>(s)] = worst;
        if (worst > 0) steps.push_back(s);  // zero-traffic steps are elided
    }
    std::vector<std::int64_t> avail = mem_avail;
    if (avail.empty()) avail.assign(static_cast<size_t>(N), std::numeric_limits<std::int64_t>::max());
    // collectives run first, each buffer charged against the same budget
    const std::int64_t M = *std::min_element(avail.begin(), avail.end());
    for (const CommOp& c : T.collectives)
        if (c.bytes > M)
            throw exec::BudgetError(strfmt("infeasible budget: collective of %lld bytes exceeds %lld",
                                           static_cast<long long>(c.bytes), static_cast<long long>(M)));
    const std::vector<std::vector<int>> stages = memory_aware_chunk(steps, T.step_cost, avail, &T.budget);
    for (const std::vector<int>& st : stages) {
        Stage S;
        S.steps = st;
        S.ranks.resize(static_cast<size_t>(N));
        for (int i = 0; i < N; ++i)
            for (int s : st) {
                RankStep rs;
                rs.step = s;
                rs.peer = xor_peer(i, s, N);
                if (rs.peer >= 0 && (bytes_of(i, rs.peer) + bytes_of(rs.peer, i)) > 0) {
                    for (int dir = 0; dir < 2; ++dir) {
                        PeerBuffer& B = dir == 0 ? rs.send : rs.recv;
                        B.peer = rs.peer;
                        const auto& list = dir == 0 ? pair[static_cast<size_t>(i)][static_cast<size_t>(rs.peer)]
                                                    : pair[static_cast<size_t>(rs.peer)][static_cast<size_t>(i)];
                        for (std::int64_t f : list) {
                            B.frags.push_back(f);
                            B.offsets.push_back(B.bytes);
                            B.bytes += T.frags[static_cast<size_t>(f)].bytes;
                        }
                    }
                } else {
                    rs.peer = -1;
                }
                S.ranks[static_cast<size_t>(i)].push_back(std::move(rs));
            }
        for (int s : st) S.mem_cost += T.step_cost[static_cast<size_t>(s)];
        T.stages.push_back(std::move(S));
    }
    return T;
}

std::string dump_schedule(const core::PlanCore& P, const TransitionSchedule& T) {
    std::string out = strfmt("# schedule N=%d budget=%lld stages=%zu collectives=%zu\n", T.N,
                             static_cast<long long>(T.budget), T.stages.size(), T.collectives.size());
    auto line = [&](const Fragment& f) {
        std::string region;
        if (f.tensor < 0) {
            region = strfmt("[%lld:%lld]", static_cast<long long>(f.lo[0]), static_cast<long long>(f.hi[0]));
        } else {
            const int nd = static_cast<int>(P.space->entries()[static_cast<size_t>(f.tensor)].spec.shape.size());
            region = "[";
            for (int d = 0; d < nd; ++d)
                region += strfmt(d ? ",%lld:%lld" : "%lld:%lld", static_cast<long long>(f.lo[d]), static_cast<long long>(f.hi[d]));
            region += "]";
        }
        return strfmt("%s %s %s src=%d dst=%d bytes=%lld", to_string(static_cast<StateKind>(f.kind)),
                      f.tensor < 0 ? "-" : P.space->entries()[static_cast<size_t>(f.tensor)].spec.tensor_id.c_str(),
                      region.c_str(), f.src_rank, f.dst_rank, static_cast<long long>(f.bytes));
    };
    static const char* names[] = {"p2p", "broadcast", "scatter", "gather"};
    for (const CommOp& c : T.collectives) {
        std::string parts;
        for (size_t i = 0; i < c.participants.size(); ++i) parts += strfmt(i ? ",%d" : "%d", c.participants[i]);
        out += strfmt("collective %s root=%d participants=%s bytes=%lld\n", names[static_cast<int>(c.kind)], c.root,
                      parts.c_str(), static_cast<long long>(c.bytes));
        for (std::int64_t f : c.frags) out += "  " + line(T.frags[static_cast<size_t>(f)]) + "\n";
    }
    for (size_t k = 0; k < T.stages.size(); ++k) {
        const Stage& S = T.stages[k];
        for (size_t si = 0; si < S.steps.size(); ++si)
            for (int i = 0; i < T.N; ++i) {
                const RankStep& rs = S.ranks[static_cast<size_t>(i)][si];
                if (rs.peer < 0) continue;
                for (size_t q = 0; q < rs.send.frags.size(); ++q)
                    out += strfmt("stage %zu step %d dev %d->%d off=%lld ", k, rs.step, i, rs.peer,
                                  static_cast<long long>(rs.send.offsets[q])) +
                           line(T.frags[static_cast<size_t>(rs.send.frags[q])]) + "\n";
            }
    }
    return out;
}

}  // namespace sched
}  // namespace reshard
