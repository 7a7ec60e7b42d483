"""Seeded random-init parameters (input generator; no method arithmetic).

Glorot-uniform weights, zero biases.  Per HGNN layer l:
W_rel [R, K_l, D] (per-relation projection, reading C3), W_root [T, K_l, D]
(RGCN self-connection, reading C4; None for RGAT), bias [T, D], att [R, 2, D]
(RGAT a_src | a_dst per relation, heads concatenated, reading C6; None for
RGCN); classifier Wc [D, C], bc [C].
"""
from __future__ import annotations

import numpy as np

from .configs import SEED, WorkloadConfig
from .graph import glorot


def make_params(cfg: WorkloadConfig, seed: int = SEED, fusion: str = "sum") -> dict:
    """fusion "han": per layer also the HAN semantic-attention parameters
    sem_W [D, A], sem_b [A], sem_q [A] with A = D (Glorot; drawn from their own
    stream, so the other parameters do not change)."""
    rng = np.random.default_rng([seed, 0xA7])
    rng_sem = np.random.default_rng([seed, 0x5E])
    T, R, D, H = cfg.num_types, cfg.num_rels, cfg.hidden, cfg.heads
    layers = []
    for l in range(cfg.num_layers):
        K = cfg.feat_dim if l == 0 else D
        lay = dict(W_rel=glorot(rng, (R, K, D), K, D),
                   W_root=glorot(rng, (T, K, D), K, D) if cfg.model == "rgcn" else None,
                   bias=np.zeros((T, D), np.float32),
                   att=glorot(rng, (R, 2, D), D // H, 1) if cfg.model == "rgat" else None)
        if fusion == "han":
            lay.update(sem_W=glorot(rng_sem, (D, D), D, D),
                       sem_b=(rng_sem.standard_normal(D) * 0.1).astype(np.float32),
                       sem_q=glorot(rng_sem, (D,), D, 1))
        layers.append(lay)
    return dict(layers=layers, Wc=glorot(rng, (D, cfg.num_classes), D, cfg.num_classes),
                bc=np.zeros(cfg.num_classes, np.float32))
