"""CPU oracle of the HiFuse hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2408_08490_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``hifuse_oracle.c`` (plain C, fp64, relation
by relation, each function citing the PAPER.md passage it follows); this module
only marshals numpy arrays through ctypes and composes the layers
(``oracle.model``).

Parity status: every function is pinned by tests/test_oracle_*.py (see
DESIGN.md §Oracle pins); the semantic readings C1-C8 themselves are "parity
unpinned by the paper" (the paper prints no equations for RGCN/RGAT).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hifuse_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

AGG = {"sum": 0, "mean": 1, "gat": 2, "gat_xrel": 3, "gat_mul": 4}


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-fopenmp", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        _lib.oracle_build.restype = ctypes.c_int
        _lib.oracle_set_threads(1)
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's parallel loops (results are bit-identical
    for any count: single writer per output, serial summation order)."""
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Shape:
    """Host metadata of one layer (types, relations, per-type counts)."""

    def __init__(self, rel_src, rel_dst, n_src, n_dst, num_edges):
        self.rel_src = _i32(rel_src)
        self.rel_dst = _i32(rel_dst)
        self.n_src = _i32(n_src)
        self.n_dst = _i32(n_dst)
        self.T = len(self.n_src)
        self.R = len(self.rel_src)
        self.N = int(num_edges)
        self.rows = int(sum(int(self.n_dst[t]) for t in self.rel_dst))
        self.S = int(sum(int(self.n_src[t]) for t in self.rel_src))
        self.src_rows = int(self.n_src.sum())
        self.dst_rows = int(self.n_dst.sum())

    @classmethod
    def of(cls, blk, rel_src, rel_dst):
        return cls(rel_src, rel_dst, blk.n_src, blk.n_dst, blk.num_edges)

    def head(self):
        return (self.T, self.R, _p(self.rel_src), _p(self.rel_dst), _p(self.n_src), _p(self.n_dst))


def build(shape: Shape, blk, edge_type):
    """O1: Alg. 2 selection + merged CSR/CSC (see hifuse_oracle.c)."""
    N = shape.N
    src, dst = _i32(blk.src_local), _i32(blk.dst_local)
    eid = np.ascontiguousarray(blk.edge_id, dtype=np.int64)
    et = _i32(edge_type)
    out = dict(rel_row_off=np.zeros(shape.R + 1, np.int32),
               row_ptr=np.zeros(shape.rows + 1, np.int32),
               col=np.zeros(N, np.int32), eperm=np.zeros(N, np.int32),
               rel_y_off=np.zeros(shape.R + 1, np.int32),
               y_src=np.full(max(N, 1), -1, np.int32),
               col_ptr=np.zeros(max(N, 1) + 1, np.int32),
               csc_pos=np.zeros(N, np.int32), csc_row=np.zeros(N, np.int32),
               slot_y=np.zeros(max(shape.S, 1), np.int32))
    U = ctypes.c_int32(0)
    st = lib().oracle_build(
        *shape.head(), ctypes.c_int64(N), _p(src), _p(dst), _p(eid), _p(et),
        ctypes.c_int64(len(et)),
        _p(out["rel_row_off"]), _p(out["row_ptr"]), _p(out["col"]), _p(out["eperm"]),
        _p(out["rel_y_off"]), _p(out["y_src"]), _p(out["col_ptr"]), _p(out["csc_pos"]),
        _p(out["csc_row"]), _p(out["slot_y"]), ctypes.byref(U))
    out["U"] = int(U.value)
    out["status"] = int(st)
    out["y_src"] = out["y_src"][:out["U"]]
    out["col_ptr"] = out["col_ptr"][:out["U"] + 1]
    # csc_col[p] = the column u with col_ptr[u] <= p < col_ptr[u+1]; -1 past
    # the valid entries (the definition, written out)
    cc = np.full(N, -1, np.int32)
    for u in range(out["U"]):
        cc[out["col_ptr"][u]:out["col_ptr"][u + 1]] = u
    out["csc_col"] = cc
    out["slot_y"] = out["slot_y"][:shape.S]
    return out


def bf16_round(x):
    """Round to the nearest bfloat16 value, ties to even (reading C24: the BF16
    projection's operand rounding), returned as float64.  The definition
    written out on the fp32 bit pattern: keep the top 16 bits, adding half an
    ulp of the kept part plus the kept part's lowest bit (ties to even);
    values already representable (and +-0, +-inf) are unchanged.  NaN is not
    handled (never an input here)."""
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = ((u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)).astype(np.uint32)
    return u.view(np.float32).astype(np.float64).reshape(np.shape(x))


def project(shape: Shape, csr, K, D, H, X, gather_ids, W_rel, W_root, att):
    """O2: Y = X_s W_r per relation (compact rows), R0 = X_t W_root,t, RGAT scores."""
    X = _f64(X)
    gid = None if gather_ids is None else _i32(gather_ids)
    U = csr["U"]
    Y = np.zeros((max(U, 1), D))
    R0 = np.zeros((max(shape.dst_rows, 1), D))
    s_src = np.zeros((max(U, 1), H))
    s_dst = np.zeros((max(shape.rows, 1), H))
    W_rel, W_root, att = _f64(W_rel), _f64(W_root), _f64(att)
    lib().oracle_project(*shape.head(), K, D, H, _p(X), _p(gid), _p(csr["rel_y_off"]),
                         _p(_i32(csr["y_src"]) if U else np.zeros(1, np.int32)),
                         _p(W_rel), _p(W_root), _p(att), _p(Y), _p(R0), _p(s_src), _p(s_dst))
    return dict(Y=Y[:U], R0=R0[:shape.dst_rows], s_src=s_src[:U], s_dst=s_dst[:shape.rows])


def aggregate_fwd(shape: Shape, blk, edge_type, csr, agg, D, H, Y, s_src=None, s_dst=None,
                  slope=0.2):
    """O3: Alg. 1 merged aggregation; returns Z [rows, D], deg [rows], alpha [N, H]."""
    N = shape.N
    Z = np.zeros((max(shape.rows, 1), D))
    deg = np.zeros(max(shape.rows, 1))
    alpha = np.zeros((max(N, 1), H)) if AGG[agg] >= 2 else None
    Yc = _f64(Y) if len(Y) else np.zeros((1, D))
    ss = _f64(s_src) if s_src is not None and len(s_src) else np.zeros((1, H))
    sd = _f64(s_dst) if s_dst is not None and len(s_dst) else np.zeros((1, H))
    lib().oracle_aggregate_fwd(
        *shape.head(), ctypes.c_int64(N), _p(_i32(blk.src_local)), _p(_i32(blk.dst_local)),
        _p(np.ascontiguousarray(blk.edge_id, np.int64)), _p(_i32(edge_type)),
        ctypes.c_int64(len(edge_type)), _p(csr["rel_y_off"]),
        _p(_i32(csr["y_src"]) if csr["U"] else np.zeros(1, np.int32)),
        AGG[agg], D, H, ctypes.c_double(slope), _p(Yc), _p(ss), _p(sd), _p(Z), _p(deg),
        _p(alpha))
    return dict(Z=Z[:shape.rows], deg=deg[:shape.rows],
                alpha=None if alpha is None else alpha[:N])


def fuse(shape: Shape, D, act, Z, R0, bias, beta=None):
    """O4: H_t[i] = act(R0_t[i] + b_t + sum_{r: t(r)=t} beta_r Z[(r,i)]) (beta = 1
    unless HAN semantic-attention weights are given, O4')."""
    Hout = np.zeros((max(shape.dst_rows, 1), D))
    Zc = _f64(Z) if len(Z) else np.zeros((1, D))
    R0c = None if R0 is None else (_f64(R0) if len(R0) else np.zeros((1, D)))
    lib().oracle_fuse(shape.T, shape.R, _p(shape.rel_dst), _p(shape.n_dst), D, int(act),
                      _p(Zc), _p(R0c), _p(_f64(bias)), _p(_f64(beta)), _p(Hout))
    return Hout[:shape.dst_rows]


def sem_att(shape: Shape, D, Z, Ws, bs, q):
    """O4': HAN semantic attention; returns (w [R], beta [R])."""
    A = len(q)
    w = np.zeros(shape.R)
    beta = np.zeros(shape.R)
    Zc = _f64(Z) if len(Z) else np.zeros((1, D))
    lib().oracle_sem_att(shape.T, shape.R, _p(shape.rel_dst), _p(shape.n_dst), D, A, _p(Zc),
                         _p(_f64(Ws)), _p(_f64(bs)), _p(_f64(q)), _p(w), _p(beta))
    return w, beta


def sem_att_bwd(shape: Shape, D, Z, Ws, bs, q, beta, G):
    """O5a': adjoint of O4' + the beta-weighted sum; returns dZ [rows, D] (per
    merged row), dWs [D, A], dbs [A], dq [A]."""
    A = len(q)
    dZ = np.zeros((max(shape.rows, 1), D))
    dWs = np.zeros((D, A))
    dbs = np.zeros(A)
    dq = np.zeros(A)
    Zc = _f64(Z) if len(Z) else np.zeros((1, D))
    Gc = _f64(G) if len(G) else np.zeros((1, D))
    lib().oracle_sem_att_bwd(shape.T, shape.R, _p(shape.rel_dst), _p(shape.n_dst), D, A, _p(Zc),
                             _p(_f64(Ws)), _p(_f64(bs)), _p(_f64(q)), _p(_f64(beta)), _p(Gc),
                             _p(dZ), _p(dWs), _p(dbs), _p(dq))
    return dict(dZ=dZ[:shape.rows], dWs=dWs, dbs=dbs, dq=dq)


def fuse_bwd(shape: Shape, D, act, dH, Hv):
    """O5a: G = dH * act'(H); dbias_t = sum_i G_t[i]."""
    G = np.zeros((max(shape.dst_rows, 1), D))
    dbias = np.zeros((shape.T, D))
    dHc = _f64(dH) if len(dH) else np.zeros((1, D))
    Hc = _f64(Hv) if len(Hv) else np.zeros((1, D))
    lib().oracle_fuse_bwd(shape.T, _p(shape.n_dst), D, int(act), _p(dHc), _p(Hc), _p(G), _p(dbias))
    return G[:shape.dst_rows], dbias


def aggregate_bwd(shape: Shape, blk, edge_type, csr, agg, D, H, G, Y, s_src=None, s_dst=None,
                  slope=0.2, g_rows=False):
    """O5b: adjoint of O3. Returns dY [U,D], ds_src [U,H], ds_dst [rows,H].
    G: type-major [dst_rows, D] (dZ[(r,i)] = G_t[i]), or with g_rows the
    per-merged-row gradient dZ [rows, D] (HAN fusion)."""
    U = csr["U"]
    dY = np.zeros((max(U, 1), D))
    ds_src = np.zeros((max(U, 1), H))
    ds_dst = np.zeros((max(shape.rows, 1), H))
    Gc = _f64(G) if len(G) else np.zeros((1, D))
    Yc = _f64(Y) if len(Y) else np.zeros((1, D))
    ss = _f64(s_src) if s_src is not None and len(s_src) else np.zeros((1, H))
    sd = _f64(s_dst) if s_dst is not None and len(s_dst) else np.zeros((1, H))
    lib().oracle_aggregate_bwd(
        *shape.head(), ctypes.c_int64(shape.N), _p(_i32(blk.src_local)), _p(_i32(blk.dst_local)),
        _p(np.ascontiguousarray(blk.edge_id, np.int64)), _p(_i32(edge_type)),
        ctypes.c_int64(len(edge_type)), _p(csr["rel_y_off"]),
        _p(_i32(csr["y_src"]) if U else np.zeros(1, np.int32)), ctypes.c_int64(U),
        AGG[agg], D, H, ctypes.c_double(slope), int(bool(g_rows)), _p(Gc), _p(Yc), _p(ss), _p(sd),
        _p(dY), _p(ds_src), _p(ds_dst))
    return dict(dY=dY[:U], ds_src=ds_src[:U], ds_dst=ds_dst[:shape.rows])


def project_bwd(shape: Shape, csr, K, D, H, X, gather_ids, W_rel, W_root, att, Y, dY, G,
                ds_src, ds_dst, need_dX=True):
    """O5c: adjoint of O2 (weights, attention vectors and, if asked, inputs)."""
    X = _f64(X)
    gid = None if gather_ids is None else _i32(gather_ids)
    U = csr["U"]
    dW_rel = np.zeros((shape.R, K, D))
    dW_root = np.zeros((shape.T, K, D)) if W_root is not None else None
    datt = np.zeros((shape.R, 2, D)) if att is not None else None
    dX = np.zeros_like(X) if need_dX else None
    pad = lambda a, w: _f64(a) if a is not None and len(a) else np.zeros((1, w))
    lib().oracle_project_bwd(
        *shape.head(), K, D, H, _p(X), _p(gid), _p(csr["rel_y_off"]),
        _p(_i32(csr["y_src"]) if U else np.zeros(1, np.int32)),
        _p(_f64(W_rel)), _p(_f64(W_root)), _p(_f64(att)), _p(pad(Y, D)), _p(pad(dY, D)),
        _p(pad(G, D)), _p(pad(ds_src, H)), _p(pad(ds_dst, H)),
        _p(dX), ctypes.c_int64(X.shape[0]), _p(dW_rel), _p(dW_root), _p(datt))
    return dict(dX=dX, dW_rel=dW_rel, dW_root=dW_root, datt=datt)


def aggregate_features(shape: Shape, blk, edge_type, agg, K, X, gather_ids):
    """O6a: Alg. 1 over the raw features (aggregate-first input layer)."""
    Xagg = np.zeros((max(shape.rows, 1), K))
    gid = None if gather_ids is None else _i32(gather_ids)
    lib().oracle_aggregate_features(
        *shape.head(), ctypes.c_int64(shape.N), _p(_i32(blk.src_local)), _p(_i32(blk.dst_local)),
        _p(np.ascontiguousarray(blk.edge_id, np.int64)), _p(_i32(edge_type)),
        ctypes.c_int64(len(edge_type)), AGG[agg], K, _p(_f64(X)), _p(gid), _p(Xagg))
    return Xagg[:shape.rows]


def project_aggregated(shape: Shape, K, D, Xagg, X, gather_ids, W_rel, W_root):
    """O6b: Z[(r,i)] = Xagg[(r,i)] W_r, R0_t = X_t W_root,t."""
    Z = np.zeros((max(shape.rows, 1), D))
    R0 = np.zeros((max(shape.dst_rows, 1), D)) if W_root is not None else None
    gid = None if gather_ids is None else _i32(gather_ids)
    pad = lambda a, w: _f64(a) if len(a) else np.zeros((1, w))
    lib().oracle_project_aggregated(
        shape.T, shape.R, _p(shape.rel_dst), _p(shape.n_src), _p(shape.n_dst), K, D,
        _p(pad(Xagg, K)), _p(_f64(X)), _p(gid), _p(_f64(W_rel)), _p(_f64(W_root)), _p(Z), _p(R0))
    return dict(Z=Z[:shape.rows], R0=None if R0 is None else R0[:shape.dst_rows])


def project_aggregated_bwd(shape: Shape, K, D, Xagg, X, gather_ids, G, root=True):
    """O6c: adjoint of O6b for the weights (no dX: input layer)."""
    dW_rel = np.zeros((shape.R, K, D))
    dW_root = np.zeros((shape.T, K, D)) if root else None
    gid = None if gather_ids is None else _i32(gather_ids)
    pad = lambda a, w: _f64(a) if len(a) else np.zeros((1, w))
    lib().oracle_project_aggregated_bwd(
        shape.T, shape.R, _p(shape.rel_dst), _p(shape.n_src), _p(shape.n_dst), K, D,
        _p(pad(Xagg, K)), _p(_f64(X)), _p(gid), _p(pad(G, D)), _p(dW_rel), _p(dW_root))
    return dict(dW_rel=dW_rel, dW_root=dW_root)
