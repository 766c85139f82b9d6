"""Synthetic workloads: model specs and scenario text for the resharding path.

The scenario text format is the one `oracle/`, `oracle/_ref/ref_plan` and the
product planner (`rs_scenario_parse`) all read; see DESIGN.md §5. It carries the
reference's value structs: ModelSpec/TensorSpec (model.hpp:30-52),
ParallelConfig (parallel.hpp:28-46), WorldMap (worldmap.hpp:30-39),
Topology (topology.hpp:25-31) and PlanOptions (routing.hpp:40-44).

Tensor ids follow the reference's string ordering rules: the canonical transfer
order compares ids as strings (routing.hpp:79-84), so "l10.q" < "l2.q".
"""
from __future__ import annotations

import dataclasses
import random
from typing import List, Optional, Sequence, Tuple


@dataclasses.dataclass
class Tensor:
    """TensorSpec (model.hpp:30-44)."""
    id: str
    shape: Tuple[int, ...]
    layer: int = 0
    tp: Optional[int] = None       # tp_shard_axis
    expert: Optional[int] = None   # expert_axis (is_expert iff set)
    dtype: int = 2                 # dtype_bytes

    def numel(self) -> int:
        n = 1
        for e in self.shape:
            n *= e
        return n


@dataclasses.dataclass
class Model:
    """ModelSpec (model.hpp:48-52)."""
    name: str
    tensors: List[Tensor]
    layers: int = 1
    experts: int = 1

    def numel(self) -> int:
        return sum(t.numel() for t in self.tensors)


@dataclasses.dataclass
class Cfg:
    """ParallelConfig (parallel.hpp:28-46)."""
    dp: int = 1
    tp: int = 1
    pp: int = 1
    ep: int = 1
    zero: bool = False
    order: str = "pp-dp-tp"

    def world(self) -> int:
        return self.dp * self.tp * self.pp

    def text(self) -> str:
        return (f"dp={self.dp} tp={self.tp} pp={self.pp} ep={self.ep} "
                f"zero={int(self.zero)} order={self.order}")


@dataclasses.dataclass
class Scenario:
    model: Model
    src: Cfg
    dst: Cfg
    world_src: Optional[Sequence[int]] = None
    world_dst: Optional[Sequence[int]] = None
    nodes: int = 1
    rpn: int = 8
    grads: str = "drop"
    balance: bool = False
    scalar_words: int = 8
    seed: int = 0
    name: str = ""

    def text(self) -> str:
        out = ["version 1", f"model layers={self.model.layers} experts={self.model.experts}"]
        for t in self.model.tensors:
            s = f"tensor {t.id} {','.join(str(e) for e in t.shape)} layer={t.layer}"
            if t.tp is not None:
                s += f" tp={t.tp}"
            if t.expert is not None:
                s += f" expert={t.expert}"
            s += f" dtype={t.dtype}"
            out.append(s)
        out.append("src " + self.src.text())
        out.append("dst " + self.dst.text())
        if self.world_src is not None or self.world_dst is not None:
            ws = self.world_src if self.world_src is not None else range(self.src.world())
            wd = self.world_dst if self.world_dst is not None else range(self.dst.world())
            out.append(f"world src={','.join(map(str, ws))} dst={','.join(map(str, wd))}")
        out.append(f"topology nodes={self.nodes} rpn={self.rpn}")
        out.append(f"options grads={self.grads} balance={int(self.balance)} scalar_words={self.scalar_words}")
        out.append(f"seed {self.seed}")
        return "\n".join(out) + "\n"

    def reversed(self) -> "Scenario":
        return dataclasses.replace(self, src=self.dst, dst=self.src, world_src=self.world_dst,
                                   world_dst=self.world_src, name=self.name + ".rev")


# --------------------------------------------------------------------- models

def llama3_8b(layers: int = 32) -> Model:
    """Llama-3-8B in declaration order: 291 tensors at L=32."""
    h, kv, ffn, vocab = 4096, 1024, 14336, 128256
    ts = [Tensor("embed", (vocab, h), 0, tp=0)]
    for l in range(layers):
        p = f"l{l}."
        ts += [
            Tensor(p + "attn_norm", (h,), l),
            Tensor(p + "q", (h, h), l, tp=0),
            Tensor(p + "k", (kv, h), l, tp=0),
            Tensor(p + "v", (kv, h), l, tp=0),
            Tensor(p + "o", (h, h), l, tp=1),
            Tensor(p + "mlp_norm", (h,), l),
            Tensor(p + "gate", (ffn, h), l, tp=0),
            Tensor(p + "up", (ffn, h), l, tp=0),
            Tensor(p + "down", (h, ffn), l, tp=1),
        ]
    ts += [Tensor("final_norm", (h,), layers - 1), Tensor("lm_head", (vocab, h), layers - 1, tp=0)]
    return Model(f"llama3-8b-L{layers}", ts, layers=layers)


def llama3_70b(layers: int = 80, hidden: int = 8192, kv: int = 1024, ffn: int = 28672, vocab: int = 128256) -> Model:
    """Llama-3-70B (config 5): 723 tensors at L=80. Smaller widths give the same tensor
    list and TP axes at toy size (parity tests against the oracle's buffers)."""
    h = hidden
    ts = [Tensor("embed", (vocab, h), 0, tp=0)]
    for l in range(layers):
        p = f"l{l}."
        ts += [
            Tensor(p + "attn_norm", (h,), l),
            Tensor(p + "q", (h, h), l, tp=0),
            Tensor(p + "k", (kv, h), l, tp=0),
            Tensor(p + "v", (kv, h), l, tp=0),
            Tensor(p + "o", (h, h), l, tp=1),
            Tensor(p + "mlp_norm", (h,), l),
            Tensor(p + "gate", (ffn, h), l, tp=0),
            Tensor(p + "up", (ffn, h), l, tp=0),
            Tensor(p + "down", (h, ffn), l, tp=1),
        ]
    ts += [Tensor("final_norm", (h,), layers - 1), Tensor("lm_head", (vocab, h), layers - 1, tp=0)]
    name = f"llama3-70b-L{layers}" if h == 8192 else f"llama3-70b-shape-L{layers}-h{h}"
    return Model(name, ts, layers=layers)


def llama2_13b(layers: int = 40) -> Model:
    """LLaMA-2 13B (Table 4 ablation model): h 5120, ffn 13824, MHA, vocab 32000."""
    h, ffn, vocab = 5120, 13824, 32000
    ts = [Tensor("embed", (vocab, h), 0, tp=0)]
    for l in range(layers):
        p = f"l{l}."
        ts += [
            Tensor(p + "attn_norm", (h,), l),
            Tensor(p + "q", (h, h), l, tp=0),
            Tensor(p + "k", (h, h), l, tp=0),
            Tensor(p + "v", (h, h), l, tp=0),
            Tensor(p + "o", (h, h), l, tp=1),
            Tensor(p + "mlp_norm", (h,), l),
            Tensor(p + "gate", (ffn, h), l, tp=0),
            Tensor(p + "up", (ffn, h), l, tp=0),
            Tensor(p + "down", (h, ffn), l, tp=1),
        ]
    ts += [Tensor("final_norm", (h,), layers - 1), Tensor("lm_head", (vocab, h), layers - 1, tp=0)]
    return Model(f"llama2-13b-L{layers}", ts, layers=layers)


def table4(layers: int = 8) -> Scenario:
    """PAPER.md Table 4 ablation geometry: (TP,PP,DP) (2,8,1) -> (2,2,4), 16 ranks."""
    return Scenario(llama2_13b(layers), Cfg(tp=2, pp=8, dp=1, zero=True), Cfg(tp=2, pp=2, dp=4, zero=True),
                    rpn=16, name=f"llama2-13b-L{layers}.table4")


def qwen3_30b_a3b(layers: int = 48, experts: int = 128) -> Model:
    """Qwen3-30B-A3B-style MoE (config 4): 579 tensors at L=48."""
    h, qd, kvd, hd, eff, vocab = 2048, 4096, 512, 128, 768, 151936
    ts = [Tensor("embed", (vocab, h), 0, tp=0)]
    for l in range(layers):
        p = f"l{l}."
        ts += [
            Tensor(p + "attn_norm", (h,), l),
            Tensor(p + "q", (qd, h), l, tp=0),
            Tensor(p + "k", (kvd, h), l, tp=0),
            Tensor(p + "v", (kvd, h), l, tp=0),
            Tensor(p + "q_norm", (hd,), l),
            Tensor(p + "k_norm", (hd,), l),
            Tensor(p + "o", (h, qd), l, tp=1),
            Tensor(p + "mlp_norm", (h,), l),
            Tensor(p + "router", (experts, h), l),
            Tensor(p + "w_gate", (experts, eff, h), l, tp=1, expert=0),
            Tensor(p + "w_up", (experts, eff, h), l, tp=1, expert=0),
            Tensor(p + "w_down", (experts, h, eff), l, tp=2, expert=0),
        ]
    ts += [Tensor("final_norm", (h,), layers - 1), Tensor("lm_head", (vocab, h), layers - 1, tp=0)]
    return Model(f"qwen3-30b-a3b-L{layers}", ts, layers=layers, experts=experts)


def tiny_gpt(layers: int = 4, hidden: int = 256, vocab: int = 1024) -> Model:
    """Config 1: tiny GPT, fp32 params (dtype_bytes=4), tied embedding: 26 tensors."""
    h = hidden
    ts = [Tensor("embed", (vocab, h), 0, tp=0, dtype=4)]
    for l in range(layers):
        p = f"h{l}."
        ts += [
            Tensor(p + "ln1", (h,), l, dtype=4),
            Tensor(p + "qkv", (3 * h, h), l, tp=0, dtype=4),
            Tensor(p + "proj", (h, h), l, tp=1, dtype=4),
            Tensor(p + "ln2", (h,), l, dtype=4),
            Tensor(p + "fc1", (4 * h, h), l, tp=0, dtype=4),
            Tensor(p + "fc2", (h, 4 * h), l, tp=1, dtype=4),
        ]
    ts += [Tensor("ln_f", (h,), layers - 1, dtype=4)]
    return Model(f"tiny-gpt-L{layers}-h{h}", ts, layers=layers)


def toy_model(rng: random.Random, max_layers: int = 8, max_per_layer: int = 6, experts: int = 1,
              with_replicated: bool = True) -> Model:
    """Random toy model for campaigns (<=8 layers, <=6 tensors/layer)."""
    layers = rng.randint(1, max_layers)
    ts: List[Tensor] = []
    for l in range(layers):
        for i in range(rng.randint(1, max_per_layer)):
            kind = rng.random()
            dtype = rng.choice([2, 2, 4])
            tid = f"L{l}.t{i}"
            if experts > 1 and kind < 0.3:
                shape = (experts, rng.choice([4, 8, 12]), rng.choice([8, 16]))
                ts.append(Tensor(tid, shape, l, tp=rng.choice([1, 2]), expert=0, dtype=dtype))
            elif with_replicated and kind < 0.45:
                ts.append(Tensor(tid, (rng.choice([4, 8, 12]),), l, dtype=dtype))
            else:
                nd = rng.choice([1, 2, 2, 3])
                shape = tuple(rng.choice([8, 16, 24, 48]) for _ in range(nd))
                ts.append(Tensor(tid, shape, l, tp=rng.randrange(nd), dtype=dtype))
    return Model("toy", ts, layers=layers, experts=experts)


# ------------------------------------------------------------------ scenarios

def config2(layers: int = 32) -> Scenario:
    """BASELINE config 2 (north star): Llama-3-8B TP8 -> DP2xTP4 + ZeRO-1 (src zero=on, dp=1)."""
    return Scenario(llama3_8b(layers), Cfg(dp=1, tp=8, zero=True), Cfg(dp=2, tp=4, zero=True),
                    name=f"llama3-8b-L{layers}.tp8-to-dp2tp4-zero1")


def config1(zero: bool = False) -> Scenario:
    """BASELINE config 1: tiny GPT DP2xTP2 -> TP4 on 4 ranks (zero=True hits reference defect D2)."""
    return Scenario(tiny_gpt(), Cfg(dp=2, tp=2, zero=zero), Cfg(dp=1, tp=4, zero=zero), rpn=4,
                    name=f"tiny-gpt.dp2tp2-to-tp4{'-zero1' if zero else ''}")


def config3(layers: int = 32) -> Tuple[Scenario, Scenario]:
    """BASELINE config 3: Llama-3-8B DP8 -> DP4 (shrink) then DP4 -> DP8 (grow), ZeRO-1."""
    m = llama3_8b(layers)
    shrink = Scenario(m, Cfg(dp=8, zero=True), Cfg(dp=4, zero=True), name="llama3-8b.dp8-to-dp4")
    grow = Scenario(m, Cfg(dp=4, zero=True), Cfg(dp=8, zero=True), name="llama3-8b.dp4-to-dp8")
    return shrink, grow


def config4(layers: int = 48) -> Scenario:
    """BASELINE config 4: Qwen3-30B-A3B-style EP8 {dp8,ep8} -> EP4xTP2 {dp4,tp2,ep4}, ZeRO-1."""
    return Scenario(qwen3_30b_a3b(layers), Cfg(dp=8, ep=8, zero=True), Cfg(dp=4, tp=2, ep=4, zero=True),
                    name=f"qwen3-30b-a3b-L{layers}.ep8-to-ep4tp2")


def config5(layers: int = 80) -> Scenario:
    """BASELINE config 5: Llama-3-70B TP4xPP2 -> TP8, ZeRO-1 (reference throws: D2)."""
    return Scenario(llama3_70b(layers), Cfg(tp=4, pp=2, zero=True), Cfg(tp=8, zero=True),
                    name=f"llama3-70b-L{layers}.tp4pp2-to-tp8")


def random_cfg(rng: random.Random, model: Model, max_world: int = 16, zero: Optional[bool] = None) -> Cfg:
    """A random ParallelConfig valid for `model` (validate_config, parallel.hpp:130-146)."""
    for _ in range(1000):
        tp = rng.choice([1, 2, 4])
        pp = rng.choice([1, 2, 4])
        dp = rng.choice([1, 2, 3, 4])
        if tp * pp * dp > max_world or pp > model.layers:
            continue
        ep_choices = [e for e in (1, 2, 4) if dp % e == 0 and model.experts % e == 0]
        ep = rng.choice(ep_choices)
        if any(t.tp is not None and t.shape[t.tp] % tp for t in model.tensors):
            continue
        order = rng.choice(["pp-dp-tp", "pp-dp-tp", "dp-pp-tp", "tp-dp-pp", "pp-tp-dp"])
        return Cfg(dp=dp, tp=tp, pp=pp, ep=ep, zero=bool(rng.random() < 0.5) if zero is None else zero,
                   order=order)
    return Cfg()


def ragged_model() -> Model:
    """Edge-case model: byte rows of 1, 3, 6, 12, 14, 20 B (every alignment class) and odd
    element counts, so ZeRO shard boundaries fall mid-row."""
    return Model("ragged", [
        Tensor("emb", (12, 7), 0, tp=0, dtype=2),
        Tensor("w1", (10, 6), 0, tp=1, dtype=2),
        Tensor("n1", (7,), 0, dtype=4),
        Tensor("b1", (4, 3), 1, tp=0, dtype=1),
        Tensor("w2", (6, 5), 1, tp=0, dtype=4),
        Tensor("n2", (9,), 1, dtype=2),
        Tensor("head", (8, 10), 1, tp=0, dtype=2),
    ], layers=2)


def edge_scenarios() -> List[Scenario]:
    """Identity transitions (everything retained), ragged widths, odd ZeRO boundaries, a
    single-tensor model, join/leave world maps, migrated gradients, one scalar word."""
    m = ragged_model()
    out = [
        Scenario(m, Cfg(tp=2), Cfg(tp=2), name="edge.identity-tp2"),
        Scenario(m, Cfg(dp=2, zero=True), Cfg(dp=2, zero=True), name="edge.identity-zero"),
        Scenario(m, Cfg(tp=2), Cfg(dp=2), name="edge.ragged-tp2-to-dp2"),
        Scenario(m, Cfg(dp=2, zero=True), Cfg(tp=2, zero=True), name="edge.ragged-dp2-zero-to-tp2"),
        Scenario(m, Cfg(dp=3, zero=True), Cfg(dp=2, zero=True), name="edge.ragged-dp3-zero-to-dp2-zero"),
        Scenario(m, Cfg(pp=2), Cfg(tp=2), grads="migrate", name="edge.ragged-pp2-to-tp2-grads"),
        Scenario(Model("one", [Tensor("w", (16, 8), 0, tp=0, dtype=2)]), Cfg(tp=4), Cfg(tp=2),
                 name="edge.single-tensor"),
        Scenario(m, Cfg(dp=2, zero=True), Cfg(dp=3, zero=True), world_src=[0, 2], world_dst=[1, 2, 3],
                 name="edge.join-leave"),
        Scenario(m, Cfg(tp=2), Cfg(tp=2), scalar_words=1, name="edge.scalars-one-word"),
    ]
    return out
