"""Comparison arms for the merged hot path (SURVEY.md §8(d) "Kernel counts"
and "Extra same-box comparison arms"; north_star: "kernel count per layer
compared with an unmerged per-relation baseline").

These are MEASUREMENT baselines, not the product: they run stock PyTorch /
cuSPARSE / cuBLAS ops (the product path is libhifuse only).  Nothing here is
imported by the library or by step.py.

  (a) torch_unmerged_layer: one HGNN layer the way a PyG-style per-relation
      implementation does it (R semantic graphs,
      each with its own select / gather / scatter kernels): per relation
      `edge_type == r`, `nonzero`, `index_select` of the projected rows,
      `matmul`, `index_reduce` (mean) or the scatter-softmax of GAT, then a
      sum over relations; backward by autograd.  Counted with torch.profiler
      (CUPTI) kernels.
  (b) per_relation_aggregate: the SAME hand-written aggregation kernel
      (hifuse_aggregate_fwd) launched once per relation on the relation's row
      slice of the merged CSR (it is relation-agnostic) -- R launches instead
      of one; isolates the launch/tail cost that merging removes (PAPER.md
      line 239 "a single kernel").
  (c) cusparse_spmm: torch.sparse.mm of the merged CSR (values 1/deg) with the
      same Y, against hifuse_aggregate_fwd (RGCN mean).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch


def _kernel_count(fn, reps=1):
    """CUDA kernels launched by fn() (torch.profiler / CUPTI), memcpy and
    memset excluded."""
    from torch.profiler import profile, ProfilerActivity
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    n = 0
    for e in p.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            nm = e.name.lower()
            if "memcpy" in nm or "memset" in nm:
                continue
            n += 1
    return n / reps


def _time_ms(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def _graph_ms(fn, reps=20):
    """fn captured in a CUDA graph and replayed (no host launch overhead)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


class TorchLayerInputs:
    """Device tensors of one sampled layer block for the torch arm."""

    def __init__(self, db, l, edge_type, X, K, D, heads, model, params_l, device):
        sh = db.shapes[l]
        self.R, self.T = sh.R, sh.T
        self.rel_src, self.rel_dst = sh.rel_src, sh.rel_dst
        self.n_dst = sh.n_dst
        self.src_off = sh.type_src_off
        self.dst_off = sh.type_dst_off
        self.src = db.dev["src"][l].long()
        self.dst = db.dev["dst"][l].long()
        self.eid = db.dev["eid"][l]
        self.edge_type = edge_type
        self.X = X
        self.K, self.D, self.H, self.model = K, D, heads, model
        f = lambda a: None if a is None else torch.tensor(np.asarray(a, np.float32), device=device,
                                                          requires_grad=True)
        self.W_rel = f(params_l["W_rel"])
        self.W_root = f(params_l.get("W_root"))
        self.bias = f(params_l["bias"])
        self.att = f(params_l.get("att"))
        self.G = torch.randn(int(sh.dst_rows), D, device=device)


def torch_unmerged_layer(t: TorchLayerInputs, agg="mean", slope=0.2, act=True):
    """Forward + backward of one HGNN layer with per-relation torch ops
    (the PyG-like unmerged baseline, SURVEY.md §8(d) arm (a))."""
    X = t.X
    et = t.edge_type[t.eid]                              # EdgeType[EdgeID] (Alg. 2)
    outs = []
    for ty in range(t.T):
        n = int(t.n_dst[ty])
        xd = X[int(t.src_off[ty]):int(t.src_off[ty]) + n]
        o = t.bias[ty].expand(n, t.D)
        if t.W_root is not None:
            o = o + xd @ t.W_root[ty]
        outs.append(o)
    for r in range(t.R):
        s_ty, d_ty = int(t.rel_src[r]), int(t.rel_dst[r])
        n = int(t.n_dst[d_ty])
        if n == 0:
            continue
        idx = (et == r).nonzero().squeeze(1)             # select this semantic graph
        s = t.src.index_select(0, idx) + int(t.src_off[s_ty])
        d = t.dst.index_select(0, idx)
        msg = X.index_select(0, s) @ t.W_rel[r]          # gather + per-relation projection
        if agg == "gat":
            H, dh = t.H, t.D // t.H
            xdst = X[int(t.src_off[d_ty]):int(t.src_off[d_ty]) + n] @ t.W_rel[r]
            a_s = t.att[r, 0].view(H, dh)
            a_d = t.att[r, 1].view(H, dh)
            ss = (msg.view(-1, H, dh) * a_s).sum(-1)
            sd = (xdst.view(-1, H, dh) * a_d).sum(-1).index_select(0, d)
            e = torch.nn.functional.leaky_relu(ss + sd, slope)
            mx = torch.full((n, H), -float("inf"), device=X.device).scatter_reduce(
                0, d[:, None].expand(-1, H), e, "amax", include_self=True)
            p = torch.exp(e - mx.index_select(0, d))
            den = torch.zeros(n, H, device=X.device).index_add(0, d, p)
            alpha = p / den.index_select(0, d)
            msg = (msg.view(-1, H, dh) * alpha[:, :, None]).reshape(-1, t.D)
            out = torch.zeros(n, t.D, device=X.device).index_add(0, d, msg)
        else:
            out = torch.zeros(n, t.D, device=X.device)
            out = out.index_reduce(0, d, msg, "mean", include_self=False) if agg == "mean" \
                else out.index_add(0, d, msg)
        outs[d_ty] = outs[d_ty] + out                    # semantic fusion (sum)
    Hout = torch.cat(outs, 0)
    if act:
        Hout = torch.relu(Hout)
    (Hout * t.G).sum().backward()
    return Hout


def per_relation_aggregate(hf, csr, sh, agg, D, heads, slope, Y, s_src, s_dst, Z, stats):
    """The merged aggregation kernel launched once per relation on the row
    slice [rel_row_off[r], rel_row_off[r+1]) of the merged CSR (arm (b))."""
    views = []
    for r in range(sh.R):
        lo, hi = int(sh.rel_row_off[r]), int(sh.rel_row_off[r + 1])
        if hi == lo:
            continue
        c = hf.Csr()
        ctypes.memmove(ctypes.addressof(c), ctypes.addressof(csr.c), ctypes.sizeof(c))
        c.row_ptr = csr["row_ptr"].data_ptr() + 4 * lo
        views.append((c, lo, hi))
    H = heads

    def off(t, lo, w):
        return None if t is None else t[lo:]

    def run():
        for c, lo, hi in views:
            lib = hf.lib()
            rc = lib.hifuse_aggregate_fwd(
                ctypes.byref(c), hi - lo, hf.AGG[agg], D, H, slope, hf._ptr(Y), hf._ptr(s_src),
                hf._ptr(off(s_dst, lo, H)), hf._ptr(Z[lo:]), hf._ptr(off(stats, lo, 2 * H)),
                hf._stream(None))
            if rc != 0:
                raise hf.HifuseError("hifuse_aggregate_fwd", rc)
    return run, len(views)


def compare_layers(hf, tr, db, cfg, feat_d, et_d, params, stage_kernels):
    """All arms on one pool batch; returns the dict bench.py adds to its line
    as "merged_vs_unmerged"."""
    dev = feat_d.device
    D, H = cfg.hidden, (cfg.heads if cfg.model == "rgat" else 1)
    # run the merged step once eagerly so activations/CSR of db are current
    tr.step(db, feat_d, et_d, update=False)
    torch.cuda.synchronize()
    out = {"relations": cfg.num_rels, "layers": []}
    acts = tr.last["acts"]
    # the arms below compare aggregations over the merged Y layout: a
    # Y-numbered build (with CSC) of every layer -- the Trainer builds its
    # aggregate-first input layer in X-row mode (col = feature rows), which a
    # Y-indexed aggregation must not read
    csrs = [hf.CsrBuffers(s, dev) for s in db.shapes]
    ws = torch.empty(sum(s.build_ws for s in db.shapes) // 4 + 64, dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    hf.build_semantic_graphs(db.shapes, csrs, db.dev["src"], db.dev["dst"], db.dev["eid"], et_d,
                             ws, st, rel_edge_off=tr._et_offsets(et_d))
    torch.cuda.synchronize()
    X = feat_d[db.dev["gid"].long()]                    # layer-0 input rows (type-major batch order)
    for l, sh in enumerate(db.shapes):
        K = cfg.feat_dim if l == 0 else D
        rec = {"layer": l, "edges": sh.N, "rows": int(sh.rows)}
        fwd_names = [n for n in stage_kernels if n.endswith(f".{l}") and
                     n.split(".")[0] in ("project", "aggregate_fwd", "fuse", "aggregate_features",
                                         "project_aggregated")]
        bwd_names = [n for n in stage_kernels if n.endswith(f".{l}") and
                     n.split(".")[0] in ("fuse_bwd", "aggregate_bwd", "project_bwd",
                                         "project_aggregated_bwd")]
        rec["merged_kernels_fwd"] = int(sum(stage_kernels[n][1] for n in fwd_names))
        rec["merged_kernels_bwd"] = int(sum(stage_kernels[n][1] for n in bwd_names))
        rec["merged_us_fwd_bwd"] = round(sum(stage_kernels[n][0] for n in fwd_names + bwd_names)
                                         * 1e3, 2)
        if cfg.agg == "gat_xrel":
            # across-relation softmax: one warp per destination; the
            # per-relation arms have no per-relation meaning here
            a = acts[l]
            Yr = torch.randn(max(sh.U_max, 1), D, device=dev)
            Z = torch.empty(max(sh.rows, 1), D, device=dev)
            stats = torch.empty(max(sh.rows, 1), 2 * H, device=dev)
            merged = lambda: hf.aggregate_fwd_xrel(sh, csrs[l], D, H, tr.slope, Yr, a["s_src"],
                                                   a["s_dst"], Z, stats)
            n0 = hf.kernel_launches()
            merged()
            rec["agg_fwd_merged_launches"] = hf.kernel_launches() - n0
            rec["agg_fwd_merged_us"] = round(_graph_ms(merged) * 1e3, 2)
            out["layers"].append(rec)
            X = acts[l]["H"][:sh.dst_rows].detach()
            continue
        # (a) torch per-relation layer, fwd + bwd
        ti = TorchLayerInputs(db, l, et_d, X.detach(), K, D, H, cfg.model, params["layers"][l],
                              dev)
        act = l < cfg.num_layers - 1
        fn = lambda: torch_unmerged_layer(ti, cfg.agg, tr.slope, act)
        try:
            rec["torch_unmerged_kernels_fwd_bwd"] = _kernel_count(fn)
        except Exception as e:                      # profiler unavailable: say so
            rec["torch_unmerged_kernels_fwd_bwd"] = f"unavailable: {type(e).__name__}"
        rec["torch_unmerged_us_fwd_bwd"] = round(_time_ms(fn, 10) * 1e3, 2)
        # (b) / merged aggregation: same kernel, one launch vs one per relation,
        # both replayed from CUDA graphs; random Y of the merged layout
        Yr = torch.randn(max(sh.U_max, 1), D, device=dev)
        a = acts[l]
        Z = torch.empty(max(sh.rows, 1), D, device=dev)
        ssrc = a["s_src"] if cfg.agg == "gat" else None
        sdst = a["s_dst"] if cfg.agg == "gat" else None
        stats = torch.empty(max(sh.rows, 1), 2 * H, device=dev) if cfg.agg == "gat" else None
        merged = lambda: hf.aggregate_fwd(csrs[l], sh.rows, cfg.agg, D, H, tr.slope, Yr, ssrc,
                                          sdst, Z, stats)
        n0 = hf.kernel_launches()
        merged()
        rec["agg_fwd_merged_launches"] = hf.kernel_launches() - n0
        rec["agg_fwd_merged_us"] = round(_graph_ms(merged) * 1e3, 2)
        Zm = Z.clone()
        per, nrel = per_relation_aggregate(hf, csrs[l], sh, cfg.agg, D, H, tr.slope, Yr, ssrc,
                                           sdst, Z, stats)
        n0 = hf.kernel_launches()
        per()
        rec["agg_fwd_per_relation_launches"] = hf.kernel_launches() - n0
        rec["agg_fwd_per_relation_us"] = round(_graph_ms(per) * 1e3, 2)
        torch.cuda.synchronize()
        rec["per_relation_equals_merged"] = bool(torch.equal(Z, Zm))
        # (c) cuSPARSE SpMM on the merged CSR (RGCN mean)
        if cfg.agg in ("mean", "sum"):
            rp = csrs[l]["row_ptr"][:sh.rows + 1].long()
            nnz = int(rp[-1].item())
            col = csrs[l]["col"][:nnz].long()
            deg = (rp[1:] - rp[:-1]).clamp(min=1).float()
            rowid = torch.repeat_interleave(torch.arange(sh.rows, device=dev), rp[1:] - rp[:-1])
            vals = (1.0 / deg)[rowid] if cfg.agg == "mean" else torch.ones(nnz, device=dev)
            A = torch.sparse_csr_tensor(rp, col, vals, size=(sh.rows, Yr.shape[0]))
            sp = lambda: torch.sparse.mm(A, Yr)
            rec["cusparse_spmm_us"] = round(_time_ms(sp, 20) * 1e3, 2)
            torch.cuda.synchronize()
            rec["cusparse_max_abs_diff"] = float((sp() - Zm[:sh.rows]).abs().max().item()) \
                if sh.rows else 0.0
        out["layers"].append(rec)
        X = acts[l]["H"][:sh.dst_rows].detach()
    return out
