"""Workload shapes of the five BASELINE.json configurations.

Seeded-input module shared by the oracle side and the CUDA side. It holds NO
arithmetic of the method (no build, projection, aggregation or fusion): only
the shapes, the seeds and the random-number recipe of the synthetic inputs.

Shapes are the HGB/OGB statistics recorded in SURVEY.md §8(d) (the paper's own
datasets, PAPER.md Table `table:dataset` lines 376-379, are RDF graphs that the
GPU box cannot download).  Relations are listed as (name, src_type, dst_type,
edge_count); a relation named ``rev_*`` mirrors the forward relation before it
(same edges, endpoints swapped).  ``sym`` relations hold both directions of
their edges (ogbn-mag ``cites``, PyG ``ToUndirected`` convention).
"""
from __future__ import annotations

from dataclasses import dataclass, field

SEED = 2408  # global seed, SURVEY.md §8(d)


@dataclass(frozen=True)
class RelSpec:
    name: str
    src: int
    dst: int
    edges: int          # edges generated for this relation (before mirroring)
    mirror_of: int = -1  # >=0: this relation is the reverse of relation `mirror_of`
    sym: bool = False   # edges stored in both directions inside this relation


@dataclass(frozen=True)
class WorkloadConfig:
    key: str
    description: str
    type_names: tuple
    type_counts: tuple
    rels: tuple
    target_type: int
    num_classes: int
    feat_dim: int        # K of layer 0
    hidden: int          # D of every HGNN layer
    heads: int           # 1 for RGCN
    model: str           # "rgcn" | "rgat"
    batch_size: int
    fanout: tuple        # per hop, hop 1 (seed neighbourhood) first
    zipf: float = 0.8
    agg: str = "mean"    # RGCN reducer (reading C1); "gat" for RGAT

    @property
    def num_layers(self) -> int:
        return len(self.fanout)

    @property
    def num_types(self) -> int:
        return len(self.type_counts)

    @property
    def num_rels(self) -> int:
        return len(self.rels)


def _mirror(rels):
    """Append the reverse of every forward relation (HGB convention)."""
    out = list(rels)
    n = len(rels)
    for i in range(n):
        r = rels[i]
        out.append(RelSpec("rev_" + r.name, r.dst, r.src, r.edges, mirror_of=i))
    return tuple(out)


def _freebase_rels(n_fwd=18):
    # 18 forward relations over distinct ordered type pairs, round-robin
    # ("round-robin over type pairs"), then 18 reverses;
    # 1,057,688 edges split evenly over the 36 relations.  Other n_fwd: the
    # supplementary R-sweep, same total edge count.
    total = 1_057_688
    per = total // (2 * n_fwd)
    fwd = []
    for k in range(n_fwd):
        s = k % 8
        t = (s + 1 + k // 8) % 8
        fwd.append(RelSpec(f"r{k}", s, t, per))
    return _mirror(tuple(fwd))


CONFIGS = {
    "acm": WorkloadConfig(
        key="acm",
        description="ACM-shaped tiny heterograph, 1-layer RGCN, 128 seeds, fanout [10], fp32",
        type_names=("paper", "author", "subject"),
        type_counts=(3025, 5959, 56),
        rels=_mirror((RelSpec("writes", 1, 0, 9949), RelSpec("about", 2, 0, 3025))),
        target_type=0, num_classes=3, feat_dim=64, hidden=64, heads=1,
        model="rgcn", batch_size=128, fanout=(10,)),
    "dblp": WorkloadConfig(
        key="dblp",
        description="DBLP-shaped heterograph, 2-layer RGCN, batch 1024, fanout [10,10]",
        type_names=("author", "paper", "term", "venue"),
        type_counts=(4057, 14328, 7723, 20),
        rels=_mirror((RelSpec("ap", 0, 1, 19645), RelSpec("tp", 2, 1, 85810),
                      RelSpec("vp", 3, 1, 14328))),
        target_type=0, num_classes=4, feat_dim=128, hidden=128, heads=1,
        model="rgcn", batch_size=1024, fanout=(10, 10)),
    "imdb": WorkloadConfig(
        key="imdb",
        description="IMDB-shaped heterograph, 2-layer RGAT (8 heads), batch 1024, fanout [10,10]",
        type_names=("movie", "director", "actor", "keyword"),
        type_counts=(4932, 2393, 6124, 7971),
        rels=_mirror((RelSpec("dm", 1, 0, 4932), RelSpec("am", 2, 0, 14779),
                      RelSpec("km", 3, 0, 23610))),
        target_type=0, num_classes=5, feat_dim=128, hidden=128, heads=8,
        model="rgat", batch_size=1024, fanout=(10, 10), agg="gat"),
    "mag": WorkloadConfig(
        key="mag",
        description="ogbn-mag-shaped synthetic (1.94M vertices, 4 types, 7 relations incl. "
                    "reverse, ~42M stored edges, feat 128), 2-layer RGCN, batch 1024, fanout [25,20]",
        type_names=("paper", "author", "institution", "field"),
        type_counts=(736_389, 1_134_649, 8_740, 59_965),
        rels=(RelSpec("writes", 1, 0, 7_145_660),
              RelSpec("cites", 0, 0, 5_416_271, sym=True),
              RelSpec("has_topic", 0, 3, 7_505_078),
              RelSpec("affiliated", 1, 2, 1_043_998),
              RelSpec("rev_writes", 0, 1, 7_145_660, mirror_of=0),
              RelSpec("rev_has_topic", 3, 0, 7_505_078, mirror_of=2),
              RelSpec("rev_affiliated", 2, 1, 1_043_998, mirror_of=3)),
        target_type=0, num_classes=349, feat_dim=128, hidden=128, heads=1,
        model="rgcn", batch_size=1024, fanout=(25, 20)),
    "freebase": WorkloadConfig(
        key="freebase",
        description="Freebase-shaped many-relation stress (8 types, 36 relations, feat 64), "
                    "2-layer RGAT (8 heads), batch 2048, fanout [10,10]",
        type_names=tuple(f"t{i}" for i in range(8)),
        type_counts=(40_402, 19_427, 82_351, 1_025, 17_641, 9_368, 2_731, 7_153),
        rels=_freebase_rels(),
        target_type=0, num_classes=7, feat_dim=64, hidden=64, heads=8,
        model="rgat", batch_size=2048, fanout=(10, 10), agg="gat"),
}

CONFIG_ORDER = ("acm", "dblp", "imdb", "mag", "freebase")


def freebase_sweep(num_rels: int, model: str = "rgat") -> WorkloadConfig:
    """Freebase-shaped graph with ``num_rels`` relations (even: forward +
    reverse) and the same total edge count; the supplementary R-sweep of
    SURVEY.md §8(d) (kernels per layer vs relation count)."""
    import dataclasses
    if num_rels % 2:
        raise ValueError("num_rels must be even (forward + reverse relations)")
    base = CONFIGS["freebase"]
    extra = {} if model == "rgat" else dict(model="rgcn", agg="mean", heads=1)
    what = "RGAT (8 heads)" if model == "rgat" else "RGCN (mean)"
    return dataclasses.replace(
        base, key=f"freebase_r{num_rels}_{model}", rels=_freebase_rels(num_rels // 2),
        description=f"Freebase-shaped R-sweep ({num_rels} relations, 8 types, feat 64), "
                    f"2-layer {what}, batch 2048, fanout [10,10]", **extra)
