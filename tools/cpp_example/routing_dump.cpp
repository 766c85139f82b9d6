// A C++ caller of the reference's routing API, unchanged except for the include path:
// the tiny GPT of BASELINE config 1 (DP2xTP2 -> TP4), planned with plan_parameters +
// plan_optimizer + plan_scalars + resolve_peers, printed with format_transfer.
//
//   g++ -std=c++20 -I paper_2605_18815_b200/csrc routing_dump.cpp
//       -L paper_2605_18815_b200/_lib -lreshard_b200 -o routing_dump
#include <cstdio>
#include <string>

#include "reshard/routing.hpp"

using namespace reshard;

int main(int argc, char** argv) {
    const bool zero = argc > 1 && std::string(argv[1]) == "zero";
    const int L = 4, h = 256, vocab = 1024;
    ModelSpec m;
    m.num_layers = L;
    auto add = [&](std::string id, std::vector<std::int64_t> shape, int layer, int tp_axis) {
        TensorSpec t;
        t.tensor_id = std::move(id);
        t.shape = std::move(shape);
        t.layer = layer;
        if (tp_axis >= 0) t.tp_shard_axis = tp_axis;
        t.dtype_bytes = 4;
        m.tensors.push_back(t);
    };
    add("embed", {vocab, h}, 0, 0);
    for (int l = 0; l < L; ++l) {
        const std::string p = "h" + std::to_string(l) + ".";
        add(p + "ln1", {h}, l, -1);
        add(p + "qkv", {3 * h, h}, l, 0);
        add(p + "proj", {h, h}, l, 1);
        add(p + "ln2", {h}, l, -1);
        add(p + "fc1", {4 * h, h}, l, 0);
        add(p + "fc2", {h, 4 * h}, l, 1);
    }
    add("ln_f", {h}, L - 1, -1);
    try {
        const ModelSpace space = build_model_space(m);
        ParallelConfig src, dst;
        src.dp = 2, src.tp = 2, src.zero_enabled = zero;
        dst.tp = 4, dst.zero_enabled = zero;
        RoutingPlan plan = plan_parameters(space, src, dst, WorldMap::identity(4, 4));
        plan_optimizer(space, plan);
        plan_scalars(plan);
        Topology topo;
        topo.num_nodes = 1;
        topo.ranks_per_node = 4;
        resolve_peers(plan, topo);
        for (const SliceTransfer& t : plan.transfers) std::printf("%s\n", format_transfer(t).c_str());
        std::printf("# transfers=%zu bytes_moved=%lld bytes_retained=%lld\n", plan.transfers.size(),
                    static_cast<long long>(plan.bytes_moved()), static_cast<long long>(plan.bytes_retained(space)));
    } catch (const ConfigError& e) {
        std::printf("# error: %s\n", e.what());
        return 2;
    }
    return 0;
}
