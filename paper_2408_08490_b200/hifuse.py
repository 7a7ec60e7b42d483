"""Thin ctypes binding of libhifuse.so (include/hifuse.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  Tensors are torch CUDA tensors (torch provides device memory and
streams); host metadata are numpy int32 arrays.  There is no CPU fallback:
importing this module on a machine without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhifuse.so")

AGG = {"sum": 0, "mean": 1, "gat": 2, "gat_xrel": 3, "gat_mul": 4}
ACT = {"none": 0, "relu": 1}
LAYOUT_COMPACT = 1
PREC = {"fp32": 0, "tf32": 1, "bf16": 2}
STATUS = {0: "ok", 1: "invalid argument", 2: "alignment", 3: "unsupported", 4: "workspace",
          5: "cuda"}


class HifuseError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)} ({code})")
        self.code = code


class LayerShape(ctypes.Structure):
    _fields_ = [("num_types", ctypes.c_int32), ("num_rels", ctypes.c_int32),
                ("rel_src_type_h", ctypes.c_void_p), ("rel_dst_type_h", ctypes.c_void_p),
                ("n_src_h", ctypes.c_void_p), ("n_dst_h", ctypes.c_void_p),
                ("num_edges", ctypes.c_int64)]


class Csr(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("rel_row_off", "row_ptr", "col", "eperm", "rel_y_off", "y_src", "col_ptr",
                 "csc_pos", "csc_row", "csc_col", "slot_y", "U_dev", "x_gather")]


class GraphCsc(ctypes.Structure):
    _fields_ = [("num_types", ctypes.c_int32), ("num_rels", ctypes.c_int32),
                ("rel_src_type_h", ctypes.c_void_p), ("rel_dst_type_h", ctypes.c_void_p),
                ("type_count_h", ctypes.c_void_p), ("in_ptr_off_h", ctypes.c_void_p),
                ("d_in_ptr", ctypes.c_void_p), ("d_in_src", ctypes.c_void_p),
                ("d_in_eid", ctypes.c_void_p)]


class Block(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("src_local", "dst_local", "edge_id", "src_gid", "counts", "gather_ids")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make -C paper_2408_08490_b200` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, f32, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                 ctypes.c_size_t)
        sig = {
            "hifuse_csr_sizes": [vp, i32, vp, vp, vp, vp],
            "hifuse_build_semantic_graphs": [vp, i32, vp, vp, vp, vp, i64, vp, i32, vp, vp, sz, vp,
                                             vp],
            "hifuse_edge_type_offsets": [vp, i64, i32, vp, vp, vp],
            "hifuse_project_ws_bytes": [vp, i32, i32, i32],
            "hifuse_project": [vp, vp, i32, i32, i32, i32, i32, vp, i64, vp, vp, vp, vp, vp, vp,
                               vp, vp, vp, sz, vp],
            "hifuse_project_y16": [vp, vp, i32, i32, i32, i32, vp, i64, vp, vp, vp, vp, vp, vp, sz,
                                   vp],
            "hifuse_aggregate_fwd": [vp, i64, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp],
            "hifuse_aggregate_fwd_xrel": [vp, vp, i32, i32, f32, vp, vp, vp, vp, vp, vp],
            "hifuse_semantic_fuse": [vp, i32, i32, vp, vp, vp, vp, vp],
            "hifuse_fuse_bwd_ws_bytes": [vp, i32],
            "hifuse_semantic_fuse_bwd": [vp, i32, i32, vp, vp, vp, vp, vp, sz, vp],
            "hifuse_semantic_fuse_bwd_bias": [vp, i32, vp, vp, vp, sz, vp],
            "hifuse_aggregate_fuse_ws_bytes": [vp],
            "hifuse_aggregate_fuse_fwd": [vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp],
            "hifuse_aggregate_bwd_ws_bytes": [vp, i32, i32],
            "hifuse_aggregate_bwd": [vp, vp, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp,
                                     vp, sz, vp],
            "hifuse_aggregate_bwd_scored": [vp, vp, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp,
                                            vp, vp, vp, sz, vp],
            "hifuse_aggregate_bwd_rows": [vp, vp, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp,
                                          vp, vp, vp, sz, vp],
            "hifuse_project_bwd_scored": [vp, vp, i32, i32, i32, i32, i32, vp, i64, vp, vp, vp, vp,
                                          vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp],
            "hifuse_project_bwd_ws_bytes": [vp, i32, i32, i32],
            "hifuse_project_bwd": [vp, vp, i32, i32, i32, i32, i32, vp, i64, vp, vp, vp, vp, vp,
                                   vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp],
            "hifuse_aggregate_features_ws_bytes": [vp],
            "hifuse_aggregate_features_fwd": [vp, vp, i32, i32, vp, i64, vp, vp, vp, sz, vp],
            "hifuse_feature_cols": [vp, vp, vp, vp, vp],
            "hifuse_aggregate_features_cols": [vp, vp, i32, i32, vp, i64, vp, vp, vp],
            "hifuse_project_aggregated": [vp, vp, i32, i32, i32, vp, vp, i64, vp, vp, vp, vp, vp,
                                          vp],
            "hifuse_project_aggregated_bwd_ws_bytes": [vp, i32, i32],
            "hifuse_project_aggregated_bwd": [vp, vp, i32, i32, i32, vp, vp, i64, vp, vp, vp, vp,
                                              vp, sz, vp],
            "hifuse_xent_ws_bytes": [i32, i32, i32],
            "hifuse_linear_xent": [i32, i32, i32, vp, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp,
                                   sz, vp, vp],
            "hifuse_linear_xent_wgrad": [i32, i32, i32, vp, i64, i64, vp, vp, vp, sz, vp],
            "hifuse_sgd": [vp, vp, i64, f32, f32, vp],
            "hifuse_sample_caps": [vp, i32, vp, i64, vp, vp, vp, vp],
            "hifuse_sample_blocks": [vp, i32, vp, vp, i64, i32, ctypes.c_uint64, vp, i32, vp, vp,
                                     vp, sz, vp, vp],
            "hifuse_sample_blocks_padded": [vp, i32, vp, vp, i64, i32, ctypes.c_uint64, vp, i32,
                                            vp, vp, vp, vp, vp, sz, vp, vp],
            "hifuse_read_status": [vp, vp, vp],
            "hifuse_sem_att_ws_bytes": [vp, i32, i32],
            "hifuse_aggregate_features_cols_bf16": [vp, vp, i32, i32, vp, i64, vp, vp, vp, vp, vp],
            "hifuse_project_fuse_aggregated": [vp, vp, i32, i32, i32, i32, vp, vp, i64, vp, vp, vp,
                                               vp, vp, vp],
            "hifuse_shard_plan": [vp, i64, vp, i32, vp, vp, vp, vp],
            "hifuse_gather_words": [vp, vp, i64, i32, i64, vp, vp],
            "hifuse_scatter_words": [vp, vp, i64, i32, vp, vp],
            "hifuse_semantic_fuse_att": [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                         vp, sz, vp],
            "hifuse_semantic_fuse_att_bwd": [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                             vp, vp, vp, vp, vp, vp, sz, vp],
            "hifuse_stream_attach": [vp],
            "hifuse_stream_release": [vp],
            "hifuse_kernel_launches": [],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        for name in ("hifuse_project_ws_bytes", "hifuse_fuse_bwd_ws_bytes",
                     "hifuse_aggregate_bwd_ws_bytes", "hifuse_project_bwd_ws_bytes",
                     "hifuse_xent_ws_bytes", "hifuse_aggregate_features_ws_bytes",
                     "hifuse_project_aggregated_bwd_ws_bytes", "hifuse_sem_att_ws_bytes",
                     "hifuse_aggregate_fuse_ws_bytes"):
            getattr(L, name).restype = ctypes.c_size_t
        L.hifuse_kernel_launches.restype = ctypes.c_int64
        L.hifuse_status_string.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _check(fn, rc):
    if rc != 0:
        raise HifuseError(fn, rc)


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    # the current stream of the current device, through torch's C accessors
    # (torch.cuda.current_stream() costs ~10 us of Python per call, which
    # dominated eager steps)
    import torch
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


class Shape:
    """Host metadata of one layer; keeps the numpy arrays alive."""

    def __init__(self, rel_src, rel_dst, n_src, n_dst, num_edges):
        self.rel_src = np.ascontiguousarray(rel_src, np.int32)
        self.rel_dst = np.ascontiguousarray(rel_dst, np.int32)
        self.n_src = np.ascontiguousarray(n_src, np.int32)
        self.n_dst = np.ascontiguousarray(n_dst, np.int32)
        self.N = int(num_edges)
        self.T, self.R = len(self.n_src), len(self.rel_src)
        self.c = LayerShape(self.T, self.R, self.rel_src.ctypes.data, self.rel_dst.ctypes.data,
                            self.n_src.ctypes.data, self.n_dst.ctypes.data, self.N)
        rows, umax, S = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ws = ctypes.c_size_t()
        _check("hifuse_csr_sizes", lib().hifuse_csr_sizes(
            ctypes.byref(self.c), LAYOUT_COMPACT, ctypes.byref(rows), ctypes.byref(umax),
            ctypes.byref(S), ctypes.byref(ws)))
        self.rows, self.U_max, self.S, self.build_ws = rows.value, umax.value, S.value, ws.value
        self.src_rows = int(self.n_src.sum())
        self.dst_rows = int(self.n_dst.sum())
        self.rel_row_off = np.concatenate([[0], np.cumsum(self.n_dst[self.rel_dst])]).astype(np.int64)
        self.type_src_off = np.concatenate([[0], np.cumsum(self.n_src)]).astype(np.int64)
        self.type_dst_off = np.concatenate([[0], np.cumsum(self.n_dst)]).astype(np.int64)

    @property
    def ref(self):
        return ctypes.byref(self.c)


class CsrBuffers:
    """Device buffers of one layer's build output (torch int32 tensors)."""

    def __init__(self, shape: Shape, device, cap=None, csc=True, xrow=False):
        """xrow: X-row mode (include/hifuse.h): no Y numbering, no CSC; col
        holds each position's source row in the layer's X."""
        import torch
        cap = cap or {}
        N = max(cap.get("N", shape.N), 1)
        rows = max(cap.get("rows", shape.rows), 1)
        umax = max(cap.get("U_max", shape.U_max), 1)
        S = max(cap.get("S", shape.S), 1)
        R = cap.get("R", shape.R)
        z = lambda n: torch.empty(n, dtype=torch.int32, device=device)
        self.t = dict(rel_row_off=z(R + 1), row_ptr=z(rows + 1), col=z(N), eperm=z(N),
                      rel_y_off=z(R + 1), y_src=z(umax), col_ptr=z(umax + 1), csc_pos=z(N),
                      csc_row=z(N), csc_col=z(N), slot_y=z(S), U_dev=z(1))
        if not csc or xrow:     # transpose not built (aggregate-first input layer)
            for k in ("col_ptr", "csc_pos", "csc_row", "csc_col"):
                self.t[k] = None
        if xrow:
            for k in ("rel_y_off", "y_src", "slot_y", "U_dev"):
                self.t[k] = None
        self.c = Csr(**{k: (v.data_ptr() if v is not None else None) for k, v in self.t.items()})

    def set_x_gather(self, gather_ids):
        """X-row mode: the build maps every column through these feature-store
        row ids (col = feature row); None: col = X row."""
        self.c.x_gather = None if gather_ids is None else gather_ids.data_ptr()

    def __getitem__(self, k):
        return self.t[k]

    @property
    def ref(self):
        return ctypes.byref(self.c)


def edge_type_offsets(edge_type, num_rels, out, status, stream=None):
    """out (int64 [R+1]) = first edge id of every relation of a relation-major
    edge-type table; HIFUSE_ST_UNSORTED_TYPES in status if it is not one."""
    _check("hifuse_edge_type_offsets", lib().hifuse_edge_type_offsets(
        _ptr(edge_type), edge_type.numel(), num_rels, _ptr(out), _ptr(status), _stream(stream)))


def build_semantic_graphs(shapes, csrs, src_local, dst_local, edge_id, edge_type, ws, status,
                          stream=None, rel_edge_off=None):
    n = len(shapes)
    arr_s = (ctypes.c_void_p * n)(*[t.data_ptr() for t in src_local])
    arr_d = (ctypes.c_void_p * n)(*[t.data_ptr() for t in dst_local])
    arr_e = (ctypes.c_void_p * n)(*[t.data_ptr() for t in edge_id])
    sh = (LayerShape * n)(*[s.c for s in shapes])
    cs = (Csr * n)(*[c.c for c in csrs])
    _check("hifuse_build_semantic_graphs", lib().hifuse_build_semantic_graphs(
        sh, n, arr_s, arr_d, arr_e, _ptr(edge_type), edge_type.numel(), _ptr(rel_edge_off),
        LAYOUT_COMPACT, cs,
        _ptr(ws), ws.numel() * ws.element_size(), _ptr(status), _stream(stream)))


def project_ws_bytes(shape, K, D, heads):
    return int(lib().hifuse_project_ws_bytes(shape.ref, K, D, heads))


def project(shape, csr, K, D, heads, X, gather_ids, W_rel, W_root, att, Y, R0, s_src, s_dst, ws,
            prec="fp32", stream=None):
    _check("hifuse_project", lib().hifuse_project(
        shape.ref, csr.ref, LAYOUT_COMPACT, PREC[prec], K, D, heads, _ptr(X), X.shape[0],
        _ptr(gather_ids), _ptr(W_rel), _ptr(W_root), _ptr(att), _ptr(Y), _ptr(R0), _ptr(s_src),
        _ptr(s_dst), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def project_y16(shape, csr, K, D, X, gather_ids, W_rel, W_root, Yb, R0, ws, prec="tf32",
                stream=None):
    """hifuse_project_y16: RGCN projection with Y stored as bfloat16 (NEXT(3))."""
    import torch
    assert Yb.dtype == torch.bfloat16
    _check("hifuse_project_y16", lib().hifuse_project_y16(
        shape.ref, csr.ref, LAYOUT_COMPACT, PREC[prec], K, D, _ptr(X), X.shape[0],
        _ptr(gather_ids), _ptr(W_rel), _ptr(W_root), _ptr(Yb), _ptr(R0), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def aggregate_fwd(csr, rows, agg, D, heads, slope, Y, s_src, s_dst, Z, stats, stream=None):
    _check("hifuse_aggregate_fwd", lib().hifuse_aggregate_fwd(
        csr.ref, rows, AGG[agg], D, heads, slope, _ptr(Y), _ptr(s_src), _ptr(s_dst), _ptr(Z),
        _ptr(stats), _stream(stream)))


def aggregate_fwd_xrel(shape, csr, D, heads, slope, Y, s_src, s_dst, Z, stats, stream=None):
    """GAT with the edge-softmax across the relations of each destination."""
    _check("hifuse_aggregate_fwd_xrel", lib().hifuse_aggregate_fwd_xrel(
        shape.ref, csr.ref, D, heads, slope, _ptr(Y), _ptr(s_src), _ptr(s_dst), _ptr(Z),
        _ptr(stats), _stream(stream)))


def semantic_fuse(shape, D, act, Z, R0, bias, H, stream=None):
    _check("hifuse_semantic_fuse", lib().hifuse_semantic_fuse(
        shape.ref, D, ACT[act], _ptr(Z), _ptr(R0), _ptr(bias), _ptr(H), _stream(stream)))


def fuse_bwd_ws_bytes(shape, D):
    return int(lib().hifuse_fuse_bwd_ws_bytes(shape.ref, D))


def semantic_fuse_bwd(shape, D, act, dH, H, G, dbias, ws, stream=None):
    _check("hifuse_semantic_fuse_bwd", lib().hifuse_semantic_fuse_bwd(
        shape.ref, D, ACT[act], _ptr(dH), _ptr(H), _ptr(G), _ptr(dbias), _ptr(ws),
        0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)))


def aggregate_fuse_ws_bytes(shape):
    return int(lib().hifuse_aggregate_fuse_ws_bytes(shape.ref))


def aggregate_fuse_fwd(shape, csr, agg, D, act, Y, R0, bias, Z, H, ws, stream=None):
    """ws: int32 tensor of aggregate_fuse_ws_bytes(shape) bytes, zeroed before
    the first call (every call leaves it zeroed)."""
    _check("hifuse_aggregate_fuse_fwd", lib().hifuse_aggregate_fuse_fwd(
        shape.ref, csr.ref, AGG[agg], D, ACT[act], _ptr(Y), _ptr(R0), _ptr(bias), _ptr(Z),
        _ptr(H), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def semantic_fuse_bwd_bias(shape, D, G, dbias, ws, stream=None):
    _check("hifuse_semantic_fuse_bwd_bias", lib().hifuse_semantic_fuse_bwd_bias(
        shape.ref, D, _ptr(G), _ptr(dbias), _ptr(ws), ws.numel() * ws.element_size(),
        _stream(stream)))


def aggregate_bwd_ws_bytes(shape, agg, heads):
    return int(lib().hifuse_aggregate_bwd_ws_bytes(shape.ref, AGG[agg], heads))


def aggregate_bwd(shape, csr, agg, D, heads, slope, G, Y, s_src, s_dst, stats, dY, ds_src, ds_dst,
                  ws, stream=None):
    _check("hifuse_aggregate_bwd", lib().hifuse_aggregate_bwd(
        shape.ref, csr.ref, AGG[agg], D, heads, slope, _ptr(G), _ptr(Y), _ptr(s_src), _ptr(s_dst),
        _ptr(stats), _ptr(dY), _ptr(ds_src), _ptr(ds_dst), _ptr(ws),
        0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)))


def aggregate_bwd_scored(shape, csr, agg, D, heads, slope, G, Y, s_src, s_dst, stats, att, dY,
                         ds_src, ds_dst, ws, stream=None):
    _check("hifuse_aggregate_bwd_scored", lib().hifuse_aggregate_bwd_scored(
        shape.ref, csr.ref, AGG[agg], D, heads, slope, _ptr(G), _ptr(Y), _ptr(s_src), _ptr(s_dst),
        _ptr(stats), _ptr(att), _ptr(dY), _ptr(ds_src), _ptr(ds_dst), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def aggregate_bwd_rows(shape, csr, agg, D, heads, slope, dZ, Y, s_src, s_dst, stats, att, dY,
                       ds_src, ds_dst, ws, stream=None):
    """hifuse_aggregate_bwd_rows: per-merged-row gradient dZ [rows, D]."""
    _check("hifuse_aggregate_bwd_rows", lib().hifuse_aggregate_bwd_rows(
        shape.ref, csr.ref, AGG[agg], D, heads, slope, _ptr(dZ), _ptr(Y), _ptr(s_src),
        _ptr(s_dst), _ptr(stats), _ptr(att), _ptr(dY), _ptr(ds_src), _ptr(ds_dst), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def sem_att_ws_bytes(shape, D, A):
    return int(lib().hifuse_sem_att_ws_bytes(shape.ref, D, A))


def semantic_fuse_att(shape, D, A, act, Z, R0, bias, Ws, bs, q, beta, w, H, ws, stream=None):
    """hifuse_semantic_fuse_att: HAN semantic-attention fusion (NEXT(2))."""
    _check("hifuse_semantic_fuse_att", lib().hifuse_semantic_fuse_att(
        shape.ref, D, A, ACT[act], _ptr(Z), _ptr(R0), _ptr(bias), _ptr(Ws), _ptr(bs), _ptr(q),
        _ptr(beta), _ptr(w), _ptr(H), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def semantic_fuse_att_bwd(shape, D, A, act, dH, H, Z, Ws, bs, q, beta, G, dZ, dbias, dWs, dbs,
                          dq, ws, stream=None):
    _check("hifuse_semantic_fuse_att_bwd", lib().hifuse_semantic_fuse_att_bwd(
        shape.ref, D, A, ACT[act], _ptr(dH), _ptr(H), _ptr(Z), _ptr(Ws), _ptr(bs), _ptr(q),
        _ptr(beta), _ptr(G), _ptr(dZ), _ptr(dbias), _ptr(dWs), _ptr(dbs), _ptr(dq), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def project_bwd_ws_bytes(shape, K, D, heads):
    return int(lib().hifuse_project_bwd_ws_bytes(shape.ref, K, D, heads))


def project_bwd(shape, csr, K, D, heads, X, gather_ids, W_rel, W_root, att, Y, dY, G, ds_src,
                ds_dst, dX, dW_rel, dW_root, datt, ws, prec="fp32", stream=None):
    _check("hifuse_project_bwd", lib().hifuse_project_bwd(
        shape.ref, csr.ref, LAYOUT_COMPACT, PREC[prec], K, D, heads, _ptr(X), X.shape[0],
        _ptr(gather_ids), _ptr(W_rel), _ptr(W_root), _ptr(att), _ptr(Y), _ptr(dY), _ptr(G),
        _ptr(ds_src), _ptr(ds_dst), _ptr(dX), _ptr(dW_rel), _ptr(dW_root), _ptr(datt), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def project_bwd_scored(shape, csr, K, D, heads, X, gather_ids, W_rel, W_root, att, Y, dY, G,
                       ds_src, ds_dst, dX, dW_rel, dW_root, datt, ws, prec="fp32", stream=None):
    _check("hifuse_project_bwd_scored", lib().hifuse_project_bwd_scored(
        shape.ref, csr.ref, LAYOUT_COMPACT, PREC[prec], K, D, heads, _ptr(X), X.shape[0],
        _ptr(gather_ids), _ptr(W_rel), _ptr(W_root), _ptr(att), _ptr(Y), _ptr(dY), _ptr(G),
        _ptr(ds_src), _ptr(ds_dst), _ptr(dX), _ptr(dW_rel), _ptr(dW_root), _ptr(datt), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def aggregate_features_ws_bytes(shape):
    return int(lib().hifuse_aggregate_features_ws_bytes(shape.ref))


def aggregate_features_fwd(shape, csr, agg, K, X, gather_ids, Xagg, ws, stream=None):
    _check("hifuse_aggregate_features_fwd", lib().hifuse_aggregate_features_fwd(
        shape.ref, csr.ref, AGG[agg], K, _ptr(X), X.shape[0], _ptr(gather_ids), _ptr(Xagg),
        _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def feature_cols(shape, csr, gather_ids, col_x, stream=None):
    _check("hifuse_feature_cols", lib().hifuse_feature_cols(
        shape.ref, csr.ref, _ptr(gather_ids), _ptr(col_x), _stream(stream)))


def aggregate_features_cols(shape, csr, agg, K, X, col_x, Xagg, stream=None):
    _check("hifuse_aggregate_features_cols", lib().hifuse_aggregate_features_cols(
        shape.ref, csr.ref, AGG[agg], K, _ptr(X), X.shape[0], _ptr(col_x), _ptr(Xagg),
        _stream(stream)))


def project_aggregated(shape, csr, K, D, Xagg, X, gather_ids, W_rel, W_root, Z, R0, prec="tf32",
                       stream=None):
    _check("hifuse_project_aggregated", lib().hifuse_project_aggregated(
        shape.ref, csr.ref, PREC[prec], K, D, _ptr(Xagg), _ptr(X),
        0 if X is None else X.shape[0], _ptr(gather_ids), _ptr(W_rel), _ptr(W_root), _ptr(Z),
        _ptr(R0), _stream(stream)))


def project_aggregated_bwd_ws_bytes(shape, K, D):
    return int(lib().hifuse_project_aggregated_bwd_ws_bytes(shape.ref, K, D))


def project_aggregated_bwd(shape, csr, K, D, Xagg, X, gather_ids, G, dW_rel, dW_root, ws,
                           prec="tf32", stream=None):
    _check("hifuse_project_aggregated_bwd", lib().hifuse_project_aggregated_bwd(
        shape.ref, csr.ref, PREC[prec], K, D, _ptr(Xagg), _ptr(X),
        0 if X is None else X.shape[0], _ptr(gather_ids), _ptr(G), _ptr(dW_rel), _ptr(dW_root),
        _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def xent_ws_bytes(B, D, C):
    return int(lib().hifuse_xent_ws_bytes(B, D, C))


def linear_xent(B, D, C, H, h_row0, labels, Wc, bc, loss, dH, dWc, dbc, ws, status=None,
                stream=None):
    _check("hifuse_linear_xent", lib().hifuse_linear_xent(
        B, D, C, _ptr(H), H.shape[0], h_row0, _ptr(labels), _ptr(Wc), _ptr(bc), _ptr(loss),
        _ptr(dH), _ptr(dWc), _ptr(dbc), _ptr(ws), ws.numel() * ws.element_size(),
        _ptr(status), _stream(stream)))


def linear_xent_wgrad(B, D, C, H, h_row0, dWc, dbc, ws, stream=None):
    _check("hifuse_linear_xent_wgrad", lib().hifuse_linear_xent_wgrad(
        B, D, C, _ptr(H), H.shape[0], h_row0, _ptr(dWc), _ptr(dbc), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def sgd(param, grad, lr, grad_scale=1.0, stream=None):
    _check("hifuse_sgd", lib().hifuse_sgd(_ptr(param), _ptr(grad), param.numel(), lr, grad_scale,
                                          _stream(stream)))


def sample_caps(graph, fanout, num_seeds):
    """(edge_cap[L], src_cap[L], ws_bytes, state_ints) of hifuse_sample_caps."""
    L = len(fanout)
    fan = np.ascontiguousarray(fanout, np.int32)
    ec = np.zeros(L, np.int64)
    sc = np.zeros(L, np.int64)
    ws = ctypes.c_size_t()
    stn = ctypes.c_int64()
    _check("hifuse_sample_caps", lib().hifuse_sample_caps(
        ctypes.byref(graph), L, fan.ctypes.data, int(num_seeds), ec.ctypes.data, sc.ctypes.data,
        ctypes.byref(ws), ctypes.byref(stn)))
    return ec, sc, ws.value, stn.value


def sample_blocks(graph, fanout, seeds, target_type, key, stamp, blocks, state, ws, status,
                  stream=None, d_ctl=None):
    fan = np.ascontiguousarray(fanout, np.int32)
    arr = (Block * len(blocks))(*blocks)
    _check("hifuse_sample_blocks", lib().hifuse_sample_blocks(
        ctypes.byref(graph), len(fan), fan.ctypes.data, _ptr(seeds), seeds.numel(), target_type,
        ctypes.c_uint64(key), _ptr(d_ctl), stamp, arr, _ptr(state), _ptr(ws), ws.numel() * ws.element_size(),
        _ptr(status), _stream(stream)))


def sample_blocks_padded(graph, fanout, seeds, target_type, key, stamp, src_cap, edge_pad, blocks,
                         state, ws, status, stream=None, d_ctl=None):
    """src_cap: int64 [L, T] per-layer per-type source capacities (outer layer
    first); edge_pad: int64 [L] padded edge counts (include/hifuse.h)."""
    fan = np.ascontiguousarray(fanout, np.int32)
    cap = np.ascontiguousarray(src_cap, np.int64)
    pad = np.ascontiguousarray(edge_pad, np.int64)
    arr = (Block * len(blocks))(*blocks)
    _check("hifuse_sample_blocks_padded", lib().hifuse_sample_blocks_padded(
        ctypes.byref(graph), len(fan), fan.ctypes.data, _ptr(seeds), seeds.numel(), target_type,
        ctypes.c_uint64(key), _ptr(d_ctl), stamp, cap.ctypes.data, pad.ctypes.data, arr,
        _ptr(state), _ptr(ws), ws.numel() * ws.element_size(), _ptr(status), _stream(stream)))


def read_status(status, stream=None):
    out = ctypes.c_int32()
    _check("hifuse_read_status", lib().hifuse_read_status(_ptr(status), _stream(stream),
                                                          ctypes.byref(out)))
    return out.value


def kernel_launches():
    return int(lib().hifuse_kernel_launches())


def stream_attach(stream=None):
    """hifuse_stream_attach: create the fork/join resources of `stream` (a
    torch.cuda.Stream; default: the current stream) outside graph capture."""
    _check("hifuse_stream_attach", lib().hifuse_stream_attach(_stream(stream)))


def stream_release(stream=None):
    _check("hifuse_stream_release", lib().hifuse_stream_release(_stream(stream)))


def shard_plan(ids, n, bounds, W, counts, order, status, stream=None):
    """hifuse_shard_plan (NEXT(4)): ids grouped by owner rank."""
    _check("hifuse_shard_plan", lib().hifuse_shard_plan(
        _ptr(ids), n, _ptr(bounds), W, _ptr(counts), _ptr(order), _ptr(status), _stream(stream)))


def gather_words(src, idx, n, words, base, dst, stream=None):
    _check("hifuse_gather_words", lib().hifuse_gather_words(
        _ptr(src), _ptr(idx), n, words, base, _ptr(dst), _stream(stream)))


def scatter_words(src, idx, n, words, dst, stream=None):
    _check("hifuse_scatter_words", lib().hifuse_scatter_words(
        _ptr(src), _ptr(idx), n, words, _ptr(dst), _stream(stream)))


def project_fuse_aggregated(shape, csr, K, D, act, Xagg, X, gather_ids, W_rel, W_root, bias, H,
                            prec="tf32", stream=None):
    """hifuse_project_fuse_aggregated: the aggregate-first layer's projection
    and fusion as one GEMM per destination type (NEXT(3))."""
    _check("hifuse_project_fuse_aggregated", lib().hifuse_project_fuse_aggregated(
        shape.ref, csr.ref, PREC[prec], K, D, ACT[act], _ptr(Xagg), _ptr(X),
        X.shape[0] if X is not None else 0, _ptr(gather_ids), _ptr(W_rel), _ptr(W_root),
        _ptr(bias), _ptr(H), _stream(stream)))


def aggregate_features_cols_bf16(shape, csr, agg, K, Xb, col_x, gather_ids, Xagg, Xdst,
                                 stream=None):
    """hifuse_aggregate_features_cols_bf16: the aggregate-first input layer over
    a BF16 feature store (NEXT(3) byte diet); Xdst receives the destination rows
    in fp32 (root term)."""
    import torch
    assert Xb.dtype == torch.bfloat16
    _check("hifuse_aggregate_features_cols_bf16", lib().hifuse_aggregate_features_cols_bf16(
        shape.ref, csr.ref, AGG[agg], K, _ptr(Xb), Xb.shape[0], _ptr(col_x), _ptr(gather_ids),
        _ptr(Xagg), _ptr(Xdst), _stream(stream)))
