"""Layer composition of the oracle -- TEST INFRASTRUCTURE ONLY.

An HGNN layer is the four stages of PAPER.md lines 112-125 (semantic graph
build, feature projection, neighbour aggregation, semantic fusion), chained
outer layer first (reading C12); ReLU between layers, none after the last
(C10).  A linear classifier + mean softmax cross-entropy closes the step
(SURVEY.md M17).  Backward runs the stages' adjoints in reverse.
Everything is fp64 and calls only the C oracle plus numpy for the classifier.
"""
from __future__ import annotations

import numpy as np

from . import (Shape, build, project, aggregate_fwd, fuse, fuse_bwd, aggregate_bwd, project_bwd,
               sem_att, sem_att_bwd)


def forward(layers, edge_type, rel_src, rel_dst, X0, gather_ids, params, agg, heads,
            slope=0.2, labels=None, target_type=0):
    """Full forward. ``layers``: LayerBlocks outer first; X0: global type-major
    features; gather_ids: layer-0 source -> X0 row.  Returns a cache dict."""
    L = len(layers)
    X, gid = np.asarray(X0, np.float64), gather_ids
    cache = []
    for l, blk in enumerate(layers):
        p = params["layers"][l]
        sh = Shape.of(blk, rel_src, rel_dst)
        K = X.shape[1]
        D = p["W_rel"].shape[2]
        csr = build(sh, blk, edge_type)
        pr = project(sh, csr, K, D, heads, X, gid, p["W_rel"], p["W_root"], p["att"])
        ag = aggregate_fwd(sh, blk, edge_type, csr, agg, D, heads, pr["Y"], pr["s_src"],
                           pr["s_dst"], slope)
        act = 1 if l < L - 1 else 0
        beta = None
        if p.get("sem_W") is not None:      # HAN semantic-attention fusion (O4')
            _, beta = sem_att(sh, D, ag["Z"], p["sem_W"], p["sem_b"], p["sem_q"])
        Hh = fuse(sh, D, act, ag["Z"], pr["R0"] if p["W_root"] is not None else None, p["bias"],
                  beta=beta)
        cache.append(dict(shape=sh, csr=csr, X=X, gid=gid, proj=pr, agg=ag, H=Hh, act=act, D=D, K=K,
                          beta=beta))
        X, gid = Hh, None
    sh = cache[-1]["shape"]
    t0 = int(sh.n_dst[:target_type].sum())
    hs = X[t0:t0 + int(sh.n_dst[target_type])]
    logits = hs @ np.asarray(params["Wc"], np.float64) + np.asarray(params["bc"], np.float64)
    out = dict(cache=cache, logits=logits, hs=hs, t0=t0)
    if labels is not None:
        z = logits - logits.max(axis=1, keepdims=True)
        lse = np.log(np.exp(z).sum(axis=1))
        out["loss"] = float(np.mean(lse - z[np.arange(len(labels)), labels]))
    return out


def xent(hs, Wc, bc, labels):
    """Linear classifier + mean softmax cross-entropy on the seed rows ``hs``
    (fp64): returns loss, dlog = (softmax - onehot) / B, dWc, dbc, dhs."""
    hs = np.asarray(hs, np.float64)
    Wc = np.asarray(Wc, np.float64)
    logits = hs @ Wc + np.asarray(bc, np.float64)
    B = len(labels)
    z = logits - logits.max(axis=1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=1))
    loss = float(np.mean(lse - z[np.arange(B), labels]))
    p = np.exp(z)
    p /= p.sum(axis=1, keepdims=True)
    dlog = p.copy()
    dlog[np.arange(B), labels] -= 1.0
    dlog /= B
    return dict(loss=loss, dlog=dlog, dWc=hs.T @ dlog, dbc=dlog.sum(axis=0), dhs=dlog @ Wc.T)


def backward(fw, layers, edge_type, params, labels, agg, heads, slope=0.2):
    """Gradients of the mean cross-entropy w.r.t. every parameter."""
    logits = fw["logits"]
    B = len(labels)
    z = logits - logits.max(axis=1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(axis=1, keepdims=True)
    dlog = p.copy()
    dlog[np.arange(B), labels] -= 1.0
    dlog /= B
    grads = dict(Wc=fw["hs"].T @ dlog, bc=dlog.sum(axis=0), layers=[None] * len(layers))
    last = fw["cache"][-1]
    dH = np.zeros_like(last["H"])
    dH[fw["t0"]:fw["t0"] + B] = dlog @ np.asarray(params["Wc"], np.float64).T
    for l in range(len(layers) - 1, -1, -1):
        c = fw["cache"][l]
        pl = params["layers"][l]
        sh, D, K = c["shape"], c["D"], c["K"]
        G, dbias = fuse_bwd(sh, D, c["act"], dH, c["H"])
        sem = None
        Gz, g_rows = G, False
        if c["beta"] is not None:
            sem = sem_att_bwd(sh, D, c["agg"]["Z"], pl["sem_W"], pl["sem_b"], pl["sem_q"],
                              c["beta"], G)
            Gz, g_rows = sem["dZ"], True
        ab = aggregate_bwd(sh, layers[l], edge_type, c["csr"], agg, D, heads, Gz, c["proj"]["Y"],
                           c["proj"]["s_src"], c["proj"]["s_dst"], slope, g_rows=g_rows)
        pb = project_bwd(sh, c["csr"], K, D, heads, c["X"], c["gid"], pl["W_rel"], pl["W_root"],
                         pl["att"], c["proj"]["Y"], ab["dY"], G, ab["ds_src"], ab["ds_dst"],
                         need_dX=l > 0)
        grads["layers"][l] = dict(W_rel=pb["dW_rel"], W_root=pb["dW_root"], bias=dbias,
                                  att=pb["datt"])
        if sem is not None:
            grads["layers"][l].update(sem_W=sem["dWs"], sem_b=sem["dbs"], sem_q=sem["dq"])
        dH = pb["dX"]
    return grads
