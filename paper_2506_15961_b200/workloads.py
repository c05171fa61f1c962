"""Named verification workloads (the BASELINE.json configs) for bench.py and tests.

Every workload is a *work plan*: the plan the discharge step runs on.

* reference toy plans: committed fixtures under tests/golden/plans (produced by
  the reference's own parallelizer and shape reducer);
* Llama-3 / DeepSeek-V3 family plans: generated here (builder -> completion ->
  parallelize) at the minimal dimensions that keep every split non-degenerate
  -- the same pattern the reference's reducer produces on the toy decoder
  (batch = max(2, dp*nm), seq = 2 (a multiple of tp under sequence
  parallelism), hidden = 2, head_dim = 2, heads = 2*tp, kv_heads = tp, ffn =
  2*tp, vocab >= batch*seq and a multiple of tp). They are "shape-reduced by
  construction": the z3-based minimizer (shapes.py, exact on the toy) stalls
  on the grouped-query view products of these graphs, as the reference's does.
"""

from __future__ import annotations

import gzip
import os
from dataclasses import dataclass

from . import builder, completion
from .parallelize import ParallelConfig, parallelize
from .plan import Plan, loads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_PLANS = os.path.join(ROOT, "tests", "golden", "plans")

FIXTURES = {
    "toy-dp2tp2pp2nm2": ("dp2tp2pp2nm2.work.json.gz",
                         "reference toy decoder (2 layers), dp2 tp2 pp2 nm2, reduced by the reference"),
    "toy-tp2": ("tp2.work.json.gz", "reference toy decoder (2 layers), tp2, reduced by the reference"),
}


@dataclass(frozen=True)
class LlamaPlanSpec:
    layers: int
    tp: int
    pp: int
    dp: int
    nm: int
    sp: bool
    desc: str
    family: str = "llama3"


def reduced_llama_config(layers: int, tp: int, dp: int, nm: int, sp: bool,
                         name: str = "llama") -> builder.LlamaConfig:
    batch = max(2, dp * nm)
    seq = max(2, tp) if sp else 2
    vocab = batch * seq
    vocab += (-vocab) % tp
    return builder.LlamaConfig(layers=layers, hidden=2, heads=2 * tp, kv_heads=tp, seq=seq,
                               vocab=vocab, batch=batch, ffn=2 * tp, head_dim=2, name=name)


GENERATED = {
    # BASELINE configs[0]
    "llama-2l-tp2dp2": LlamaPlanSpec(2, tp=2, pp=1, dp=2, nm=1, sp=False,
                                     desc="2-layer Llama-style decoder, TP=2 x DP=2, shape-reduced"),
    # BASELINE configs[1] -- the N=1 bench workload
    "llama3-8b-tp4pp2dp2-sp": LlamaPlanSpec(32, tp=4, pp=2, dp=2, nm=2, sp=True,
                                            desc="Llama3-8B (32 layers, GQA) TP=4 PP=2 DP=2 nm=2 "
                                                 "with sequence parallelism, shape-reduced"),
    # BASELINE configs[3]
    "llama3-405b-tp8pp16dp2": LlamaPlanSpec(126, tp=8, pp=16, dp=2, nm=2, sp=False,
                                            desc="Llama3-405B (126 layers, GQA) TP=8 PP=16 DP=2 nm=2, "
                                                 "shape-reduced full stage sweep"),
    # BASELINE configs[4]: DeepSeek-V3 (61 layers, 3 dense) with MLA and MoE,
    # experts split over the tensor group, all_to_all token dispatch
    "deepseek-v3-tp4pp4dp2-ep": LlamaPlanSpec(61, tp=4, pp=4, dp=2, nm=2, sp=True,
                                              desc="DeepSeek-V3 (61 layers, MLA, 3 dense + 58 MoE, "
                                                   "8 routed experts + 1 shared) TP=EP=4 PP=4 DP=2 "
                                                   "nm=2 SP, shape-reduced", family="deepseek-v3"),
    # small members of the same families (tests)
    "deepseek-6l-tp4pp2dp2-ep": LlamaPlanSpec(6, tp=4, pp=2, dp=2, nm=2, sp=True,
                                              desc="6-layer DeepSeek-style decoder (3 dense + 3 MoE), "
                                                   "TP=EP=4 PP=2 DP=2 nm=2 SP", family="deepseek-v3"),
    "deepseek-2l-tp2dp2-sp": LlamaPlanSpec(2, tp=2, pp=1, dp=2, nm=1, sp=True,
                                           desc="2-layer DeepSeek-style decoder (1 dense + 1 MoE), "
                                                "TP=EP=2 DP=2 SP", family="deepseek-v3"),
    "llama-4l-tp2pp2dp2-sp": LlamaPlanSpec(4, tp=2, pp=2, dp=2, nm=2, sp=True,
                                           desc="4-layer Llama-style decoder, TP=2 PP=2 DP=2 nm=2 SP"),
    # configs[3]'s parallel shape (TP=8 PP=16 DP=2 nm=2, one layer per pipeline
    # stage) at 16 layers: the same stage programs as the 126-layer sweep,
    # small enough for the reference to verify every stage
    "llama3-405b-16l-tp8pp16dp2": LlamaPlanSpec(16, tp=8, pp=16, dp=2, nm=2, sp=False,
                                                desc="Llama3-405B-shaped (16 layers, GQA) TP=8 PP=16 "
                                                     "DP=2 nm=2, shape-reduced"),
    # mid-size MoE member the reference can finish: 3 dense + 1 MoE layer
    "deepseek-4l-tp4pp2dp2-ep": LlamaPlanSpec(4, tp=4, pp=2, dp=2, nm=2, sp=True,
                                              desc="4-layer DeepSeek-style decoder (3 dense + 1 MoE), "
                                                   "TP=EP=4 PP=2 DP=2 nm=2 SP", family="deepseek-v3"),
}
# bug-injected variants: "<workload>~<fault category>" picks one site of that
# category with a name-seeded RNG (BASELINE configs[2] on the full Llama3-8B)
FAULT_SEP = "~"
DEFAULT = "llama3-8b-tp4pp2dp2-sp"


def llama_plan(spec: LlamaPlanSpec) -> Plan:
    lc = reduced_llama_config(spec.layers, spec.tp, spec.dp, spec.nm, spec.sp)
    g = completion.complete(builder.llama_forward(lc), completion.LossSpec("mean"))
    cfg = ParallelConfig(dp=spec.dp, tp=spec.tp, pp=spec.pp, nm=spec.nm, sp=spec.sp)
    return parallelize(g, cfg, lineage_interiors=builder.toy_interiors(g))


def reduced_deepseek_config(layers: int, tp: int, dp: int, nm: int, sp: bool,
                            name: str = "deepseek") -> builder.DeepSeekConfig:
    """Minimal non-degenerate DeepSeek-V3 dimensions for a tp-way split: 2*tp
    heads and routed experts (the expert axis is what expert parallelism
    splits), 2-wide latent/rope/expert dims, the published 3 dense layers."""
    batch = max(2, dp * nm)
    seq = max(2, tp) if sp else 2
    vocab = batch * seq
    vocab += (-vocab) % tp
    return builder.DeepSeekConfig(layers=layers, dense_layers=min(3, max(1, layers - 1)),
                                  hidden=2, heads=2 * tp, head_dim=2, rope_dim=2, q_rank=2,
                                  kv_rank=2, experts=2 * tp, expert_ffn=2, ffn=2 * tp, seq=seq,
                                  vocab=vocab, batch=batch, name=name)


def deepseek_plan(spec: LlamaPlanSpec) -> Plan:
    dc = reduced_deepseek_config(spec.layers, spec.tp, spec.dp, spec.nm, spec.sp)
    g = completion.complete(builder.deepseek_forward(dc), completion.LossSpec("mean"))
    cfg = ParallelConfig(dp=spec.dp, tp=spec.tp, pp=spec.pp, nm=spec.nm, sp=spec.sp)
    return parallelize(g, cfg, lineage_interiors=builder.toy_interiors(g))


def _fixture(fname: str) -> Plan:
    with gzip.open(os.path.join(GOLDEN_PLANS, fname), "rt") as f:
        return loads(f.read())


def fault_site(plan: Plan, name: str, category: str):
    """The fault site a "<workload>~<category>" name denotes (deterministic)."""
    import random
    from .faults import list_sites
    sites = list_sites(plan, category)
    if not sites:
        raise KeyError(f"workload {name!r} has no {category!r} fault site")
    return random.Random(f"{name}{FAULT_SEP}{category}").choice(sites)


def get_workload(name: str = "default") -> tuple[str, Plan]:
    if name == "default":
        name = DEFAULT
    if FAULT_SEP in name:
        from .faults import inject
        base, category = name.split(FAULT_SEP, 1)
        desc, plan = get_workload(base)
        site = fault_site(plan, base, category)
        return (f"{name}: {desc.split(': ', 1)[-1]}; injected {category} at {site.site}",
                inject(plan, site))
    if name in FIXTURES:
        fname, desc = FIXTURES[name]
        return f"{name}: {desc}", _fixture(fname)
    if name in GENERATED:
        spec = GENERATED[name]
        if spec.family == "deepseek-v3":
            return f"{name}: {spec.desc}", deepseek_plan(spec)
        return f"{name}: {spec.desc}", llama_plan(spec)
    raise KeyError(f"unknown workload {name!r}; known: {sorted(FIXTURES) + sorted(GENERATED)}")
