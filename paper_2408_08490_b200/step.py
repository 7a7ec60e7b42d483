"""One mini-batch HGNN training step through the C ABI (Fig. 2 step
(4), line 156: forward through the four stages of every layer, backward,
parameter update).

torch supplies device memory, the stream and (for N > 1) the NCCL process
group; every arithmetic step runs in libhifuse kernels:

  hifuse_build_semantic_graphs   all layers (A1)
  per layer, outer first:        hifuse_project (A2+A3) -> hifuse_aggregate_fwd
                                 (A4) -> hifuse_semantic_fuse (A5)
  hifuse_linear_xent             classifier + loss + its gradients
  per layer, inner first:        hifuse_semantic_fuse_bwd -> hifuse_aggregate_bwd
                                 -> hifuse_project_bwd (A6)
  [dist.all_reduce of the flat gradient buffer when world_size > 1]
  hifuse_sgd                     parameter update

Parameters and gradients each live in ONE flat fp32 buffer so the data-parallel
exchange is a single NCCL all-reduce.
"""
from __future__ import annotations

import numpy as np
import torch

from . import hifuse as hf
from .dp import ParamLayout


class DeviceBatch:
    """A sampled mini-batch resident on the device (sampling is outside the
    library boundary, Fig. 2 step (1))."""

    def __init__(self, mb, rel_src, rel_dst, feat_off, target_type, device, pin=False):
        self.shapes = [hf.Shape(rel_src, rel_dst, b.n_src, b.n_dst, b.num_edges) for b in mb.layers]
        self.host = dict(
            src=[np.ascontiguousarray(b.src_local, np.int32) for b in mb.layers],
            dst=[np.ascontiguousarray(b.dst_local, np.int32) for b in mb.layers],
            eid=[np.ascontiguousarray(b.edge_id, np.int64) for b in mb.layers],
            gid=mb.gather_ids(feat_off).astype(np.int32),
            labels=np.ascontiguousarray(mb.labels, np.int32))
        self.B = len(mb.labels)
        self.slot = 0          # which CSR buffer set of the Trainer this batch uses
        self.target_type = target_type
        self.h_row0 = int(self.shapes[-1].type_dst_off[target_type])
        self.device = device
        self.dev = None
        self.pinned = None
        if pin:
            self.pinned = {k: ([torch.from_numpy(a).pin_memory() for a in v] if isinstance(v, list)
                               else torch.from_numpy(v).pin_memory())
                           for k, v in self.host.items()}
        if device is not None:
            self.to_device()

    def to_device(self, non_blocking=False):
        """Host -> device copy of the batch inputs; re-uses the device tensors
        after the first call (so captured CUDA graphs stay valid)."""
        src = self.pinned if self.pinned is not None else {
            k: ([torch.from_numpy(a) for a in v] if isinstance(v, list) else torch.from_numpy(v))
            for k, v in self.host.items()}
        if self.dev is None:
            self.dev = {k: ([t.to(self.device, non_blocking=non_blocking) for t in v]
                            if isinstance(v, list) else v.to(self.device, non_blocking=non_blocking))
                        for k, v in src.items()}
        else:
            for k, v in src.items():
                if isinstance(v, list):
                    for d, h in zip(self.dev[k], v):
                        d.copy_(h, non_blocking=non_blocking)
                else:
                    self.dev[k].copy_(v, non_blocking=non_blocking)
        return self

    def h2d_bytes(self):
        return int(sum(a.nbytes for v in self.host.values()
                       for a in (v if isinstance(v, list) else [v])))


class Trainer:
    """Owns parameters, gradients, activations and workspaces of the step."""

    def __init__(self, T, R, rel_src, rel_dst, K0, D, H, C, L, model, agg, device, lr=0.01,
                 prec="tf32", slope=0.2, order="project_first", fusion="sum", fuse_gemm=True,
                 feat_dtype="fp32", y_dtype="fp32", inner_agg_first=True):
        hf.lib()   # raises if libhifuse.so is missing (no CPU fallback)
        self.T, self.R, self.K0, self.D, self.H, self.C, self.L = T, R, K0, D, H, C, L
        self.rel_src = np.asarray(rel_src, np.int32)
        self.rel_dst = np.asarray(rel_dst, np.int32)
        self.model, self.agg, self.device, self.lr, self.prec, self.slope = (
            model, agg, device, lr, prec, slope)
        # prec "bf16": the per-relation projection (hifuse_project) runs on
        # BF16 operands (HIFUSE_PREC_BF16); the backward GEMMs and the
        # aggregate-first input layer's GEMMs take TF32 (no BF16 variant)
        if prec not in ("fp32", "tf32", "bf16"):
            raise ValueError(prec)
        self.prec_tc = "tf32" if prec == "bf16" else prec
        if fusion not in ("sum", "han"):
            raise ValueError(fusion)
        self.fusion = fusion       # "han": HAN semantic-attention fusion (NEXT(2), reading C22)
        self.layout = ParamLayout(T, R, K0, D, H, C, L, model, fusion)
        self.params = torch.zeros(self.layout.size, dtype=torch.float32, device=device)
        self.grads = torch.zeros_like(self.params)
        self.P = self.layout.views(self.params)
        self.Gd = self.layout.views(self.grads)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.loss = torch.zeros(1, dtype=torch.float32, device=device)
        self.world, self.dp_group, self._comm = 1, None, None
        self._bufs = {}
        self._views = {}
        self.heads = H if model == "rgat" else 1
        # "agg_first": the RGCN input layer aggregates raw features and then
        # projects the aggregated rows (exact by linearity; SURVEY §8(f)
        # NEXT(3)).  RGAT needs projected features for its
        # scores, so it always projects first.
        if order not in ("project_first", "agg_first"):
            raise ValueError(order)
        # (HAN fusion gives every relation its own gradient: project-first only)
        self.agg_first = (order == "agg_first" and model == "rgcn" and prec != "fp32" and
                          fusion == "sum")
        self.order = "agg_first" if self.agg_first else "project_first"
        # aggregate-first input layer: projection + fusion as one GEMM per
        # destination type (hifuse_project_fuse_aggregated, NEXT(3))
        self.fuse_gemm = bool(fuse_gemm) and self.agg_first
        # ... and the inner layers' FORWARD in the same order (their backward
        # stays project-first: RGCN's transpose SpMM, dgrad and wgrad read only
        # G, the CSC and the layer input, never Y or Z, so the two forward
        # orders feed the identical backward; exact by linearity, reading C3')
        self.agg_first_inner = bool(inner_agg_first) and self.fuse_gemm and y_dtype == "fp32"
        # NEXT(3) byte diet: BF16 storage of the input features (the
        # aggregate-first input layer reads them; its root term reads the
        # destination rows converted to fp32 by the same launch)
        if feat_dtype not in ("fp32", "bf16"):
            raise ValueError(feat_dtype)
        if feat_dtype == "bf16" and not self.agg_first:
            raise ValueError("a BF16 feature store needs the aggregate-first input layer")
        self.feat_dtype = feat_dtype
        # NEXT(3) byte diet: BF16 storage of Y (RGCN project-first layers; the
        # aggregation reads it through the BF16 gather kernel, reading C25)
        if y_dtype not in ("fp32", "bf16"):
            raise ValueError(y_dtype)
        if y_dtype == "bf16" and (model != "rgcn" or prec == "fp32" or fusion != "sum"):
            raise ValueError("BF16 Y needs the RGCN tcgen05 projection (tf32 / bf16)")
        self.y_dtype = y_dtype
        # capture streams: `_hi` (high priority) for the pipelined graphs,
        # `_cap` for the serial / per-stage graphs; the library's fork/join
        # resources of every stream that runs steps are created here, outside
        # graph capture (hifuse_stream_attach)
        self._hi = torch.cuda.Stream(device=device, priority=-1)
        self._cap = torch.cuda.Stream(device=device)
        self._head_side = torch.cuda.Stream(device=device)
        with torch.cuda.device(device):
            for s in (torch.cuda.current_stream(device), self._hi, self._cap, self._head_side):
                hf.stream_attach(s)

    def load_params(self, p):
        for l, lay in enumerate(p["layers"]):
            for k in ("W_rel", "W_root", "bias", "att", "sem_W", "sem_b", "sem_q"):
                if lay.get(k) is not None and f"{l}.{k}" in self.P:
                    self.P[f"{l}.{k}"].copy_(torch.from_numpy(np.asarray(lay[k], np.float32)))
        self.P["Wc"].copy_(torch.from_numpy(np.asarray(p["Wc"], np.float32)))
        self.P["bc"].copy_(torch.from_numpy(np.asarray(p["bc"], np.float32)))

    # ------------------------------------------------------ data parallelism
    def set_dp(self, world, group=None):
        """Data parallelism over independent mini-batches:
        the weight gradients are summed over `world` ranks with one all-reduce
        per bucket (one bucket per HGNN layer + the classifier), each issued on
        a communication stream as soon as its layer's backward has produced
        them, overlapping the backward of the layers below; the SGD applies the
        1/world factor.  With NCCL the all-reduces are capturable, so a whole
        DP step (compute + collectives + update) is one CUDA graph."""
        self.world = int(world)
        self.dp_group = group
        self._comm = torch.cuda.Stream(device=self.device) if self.world > 1 else None
        self._bk = self.layout.buckets(self.L)

    def _allreduce_op(self, key):
        """Op: the comm stream waits for everything issued so far (main and
        weight-gradient side stream) and all-reduces bucket `key`."""
        import torch.distributed as dist
        lo, hi = self._bk[key]

        def run():
            main = torch.cuda.current_stream()
            self._comm.wait_stream(main)
            self._comm.wait_stream(self._head_side)
            with torch.cuda.stream(self._comm):
                dist.all_reduce(self.grads[lo:hi], group=self.dp_group)
        return run

    def _dp_join(self):
        torch.cuda.current_stream().wait_stream(self._comm)

    # -------------------------------------------------------------- buffers
    def _buf(self, key, n, dtype=torch.float32):
        t = self._bufs.get(key)
        if t is None or t.numel() < n:
            t = torch.empty(max(int(n * 1.25), 16), dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t

    def _mat(self, key, rows, cols):
        buf = self._buf(key, max(rows, 1) * cols)
        vk = (key, rows, cols)
        v = self._views.get(vk)
        if v is None or v[0] is not buf:          # cached view (eager steps re-plan)
            v = (buf, buf[:max(rows, 1) * cols].view(max(rows, 1), cols))
            self._views[vk] = v
        return v[1]

    def _csr(self, l, shape, slot=0):
        key = f"csr{slot}.{l}"
        c = self._bufs.get(key)
        need = dict(N=shape.N, rows=shape.rows, U_max=shape.U_max, S=shape.S, R=shape.R)
        if c is None or any(need[k] > c.cap[k] for k in need):
            cap = {k: int(v * 1.25) + 1 for k, v in need.items()}
            cap["R"] = shape.R
            # the aggregate-first input layer never runs the transpose and reads
            # raw X rows: X-row build (no Y numbering, no slot scan)
            first = self.agg_first and l == 0
            c = hf.CsrBuffers(shape, self.device, cap, csc=not first, xrow=first)
            c.cap = cap
            self._bufs[key] = c
        return c

    def _zeros(self, key, n):
        """int32 buffer of >= n entries, zeroed when (re)allocated (counters
        the library leaves zeroed after every call)."""
        t = self._bufs.get(key)
        if t is None or t.numel() < n:
            t = torch.zeros(max(int(n * 1.25), 16), dtype=torch.int32, device=self.device)
            self._bufs[key] = t
        return t

    def _ws(self, nbytes, key="ws"):
        return self._buf(key, (nbytes + 3) // 4 + 64)

    def prepare_graph(self, edge_type):
        """One-time per graph (synchronises): if the edge-type table is
        relation-major, keep its R+1 offsets so that the build evaluates
        EdgeType[EdgeID] without the random table gather (include/hifuse.h)."""
        off = torch.empty(self.R + 1, dtype=torch.int64, device=self.device)
        st = torch.zeros(1, dtype=torch.int32, device=self.device)
        hf.edge_type_offsets(edge_type, self.R, off, st)
        ok = hf.read_status(st) == 0
        self._et_off = (edge_type.data_ptr(), off if ok else None)
        return ok

    def _et_offsets(self, edge_type):
        c = getattr(self, "_et_off", None)
        return c[1] if c is not None and c[0] == edge_type.data_ptr() else None

    def build_op(self, db: DeviceBatch, edge_type):
        """The semantic-graph build of ``db`` (A1) as a closure; CSR buffers
        are per batch slot and the workspace is private, so it may run on a
        side stream while another batch computes."""
        dev, shapes = db.dev, db.shapes
        csrs = [self._csr(l, s, db.slot) for l, s in enumerate(shapes)]
        wsb = self._ws(sum(s.build_ws for s in shapes), key="ws_build")   # layers built together
        off = self._et_offsets(edge_type)
        if not self.agg_first:
            return lambda: hf.build_semantic_graphs(shapes, csrs, dev["src"], dev["dst"],
                                                    dev["eid"], edge_type, wsb, self.status,
                                                    rel_edge_off=off)
        # aggregate-first input layer: X-row build whose columns are mapped
        # through the batch's gather ids, so col holds the feature-store row of
        # every CSR position (formed with the build, off the critical path)

        colxs = [self._buf(f"colx{db.slot}.{l}", max(shapes[l].N, 1), torch.int32)
                 for l in range(1, len(shapes))] if self.agg_first_inner else []

        def op():
            csrs[0].set_x_gather(dev["gid"])
            hf.build_semantic_graphs(shapes, csrs, dev["src"], dev["dst"], dev["eid"], edge_type,
                                     wsb, self.status, rel_edge_off=off)
            # inner layers (aggregate-first forward): the X row (previous
            # layer's H) of every CSR position, from their Y-numbered build
            for l, cx in enumerate(colxs, start=1):
                hf.feature_cols(shapes[l], csrs[l], None, cx)
        return op

    # ----------------------------------------------------------------- plan
    def plan(self, db: DeviceBatch, feat, edge_type, include_build=True, split_head=True):
        """The step's library calls as a list of (stage name, closure).  All
        buffers are bound here, so the closures can be run eagerly or captured
        into a CUDA graph (no allocation, no host sync inside).  split_head:
        the classifier's weight gradient runs on a side stream next to the
        layers' backward (a parallel graph branch), joined by the last op."""
        L, D, H, C = self.L, self.D, self.heads, self.C
        dev = db.dev
        shapes = db.shapes
        ops = []
        csrs = [self._csr(l, s, db.slot) for l, s in enumerate(shapes)]
        if include_build:
            ops.append(("build", self.build_op(db, edge_type)))
        acts = []
        X, gid = feat, dev["gid"]
        for l, sh in enumerate(shapes):
            K = self.K0 if l == 0 else D
            P = {k: self.P.get(f"{l}.{k}") for k in ("W_rel", "W_root", "bias", "att")}
            a = dict(X=X, gid=gid, K=K, act="relu" if l < L - 1 else "none",
                     Y=self._mat(f"Y{l}", sh.U_max, D),
                     R0=self._mat(f"R0{l}", sh.dst_rows, D) if P["W_root"] is not None else None,
                     s_src=self._mat(f"ss{l}", sh.U_max, H) if P["att"] is not None else None,
                     s_dst=self._mat(f"sd{l}", sh.rows, H) if P["att"] is not None else None,
                     Z=self._mat(f"Z{l}", sh.rows, D),
                     stats=(self._mat(f"st{l}", sh.rows, 2 * H) if self.agg.startswith("gat")
                            else None),
                     H=self._mat(f"H{l}", sh.dst_rows, D),
                     wsp=self._ws(hf.project_ws_bytes(sh, K, D, H)))
            if self.agg_first and l == 0:
                a.update(Y=None, Xagg=self._mat("Xagg0", sh.rows, K))
                # colx: the feature-store row of every CSR position, written by
                # this batch's build (X-row mode through the gather ids)
                colx = csrs[l]["col"]
                if self.feat_dtype == "bf16":
                    a.update(Xroot=self._mat("Xdst0", sh.src_rows, K), gid_root=None)
                    ops.append(("aggregate_features.0", lambda sh=sh, c=csrs[l], a=a, colx=colx:
                                hf.aggregate_features_cols_bf16(sh, c, self.agg, a["K"], a["X"],
                                                                colx, a["gid"], a["Xagg"],
                                                                a["Xroot"])))
                else:
                    a.update(Xroot=a["X"], gid_root=a["gid"])
                    ops.append(("aggregate_features.0", lambda sh=sh, c=csrs[l], a=a, colx=colx:
                                hf.aggregate_features_cols(sh, c, self.agg, a["K"], a["X"], colx,
                                                           a["Xagg"])))
                if self.fuse_gemm:
                    ops.append(("project_fuse_aggregated.0", lambda sh=sh, c=csrs[l], a=a, P=P:
                                hf.project_fuse_aggregated(sh, c, a["K"], D, a["act"], a["Xagg"],
                                                           a["Xroot"], a["gid_root"], P["W_rel"],
                                                           P["W_root"], P["bias"], a["H"],
                                                           prec=self.prec_tc)))
                else:
                    ops.append(("project_aggregated.0", lambda sh=sh, c=csrs[l], a=a, P=P:
                                hf.project_aggregated(sh, c, a["K"], D, a["Xagg"], a["Xroot"],
                                                      a["gid_root"], P["W_rel"], P["W_root"], a["Z"],
                                                      a["R0"], prec=self.prec_tc)))
                    ops.append((f"fuse.{l}", lambda sh=sh, a=a, P=P: hf.semantic_fuse(
                        sh, D, a["act"], a["Z"], a["R0"], P["bias"], a["H"])))
                acts.append(a)
                X, gid = a["H"], None
                continue
            if self.agg_first_inner and l > 0:
                # aggregate-first forward of an inner RGCN layer: the previous
                # layer's H rows aggregated, then one fused GEMM per
                # destination type (no Y, no Z); backward as project-first
                a.update(Xagg=self._mat(f"Xagg{l}", sh.rows, K))
                colx = self._buf(f"colx{db.slot}.{l}", max(sh.N, 1), torch.int32)
                ops.append((f"aggregate_features.{l}", lambda sh=sh, c=csrs[l], a=a, colx=colx:
                            hf.aggregate_features_cols(sh, c, self.agg, a["K"], a["X"], colx,
                                                       a["Xagg"])))
                ops.append((f"project_fuse_aggregated.{l}", lambda sh=sh, c=csrs[l], a=a, P=P:
                            hf.project_fuse_aggregated(sh, c, a["K"], D, a["act"], a["Xagg"],
                                                       a["X"], None, P["W_rel"], P["W_root"],
                                                       P["bias"], a["H"], prec=self.prec_tc)))
                acts.append(a)
                X, gid = a["H"], None
                continue
            if self.y_dtype == "bf16":
                yb = self._buf(f"Yb{l}", max(sh.U_max, 1) * D, torch.bfloat16)
                a["Yb"] = yb[:max(sh.U_max, 1) * D].view(max(sh.U_max, 1), D)
                ops.append((f"project.{l}", lambda sh=sh, c=csrs[l], a=a, P=P: hf.project_y16(
                    sh, c, a["K"], D, a["X"], a["gid"], P["W_rel"], P["W_root"], a["Yb"],
                    a["R0"], a["wsp"], prec=self.prec)))
                ops.append((f"aggregate_fwd.{l}", lambda sh=sh, c=csrs[l], a=a:
                            hf.aggregate_features_cols_bf16(sh, c, self.agg, D, a["Yb"], c["col"],
                                                            None, a["Z"], None)))
            else:
                ops.append((f"project.{l}", lambda sh=sh, c=csrs[l], a=a, P=P: hf.project(
                    sh, c, a["K"], D, H, a["X"], a["gid"], P["W_rel"], P["W_root"], P["att"],
                    a["Y"], a["R0"], a["s_src"], a["s_dst"], a["wsp"], prec=self.prec)))
            if self.y_dtype == "bf16":
                pass
            elif self.agg in ("sum", "mean") and self.fusion == "sum":
                # RGCN: aggregation and fusion in one launch (the last
                # relation row of a destination forms its H row)
                a["fcnt"] = self._zeros(f"fcnt{l}", hf.aggregate_fuse_ws_bytes(sh) // 4)
                ops.append((f"aggregate_fwd.{l}", lambda sh=sh, c=csrs[l], a=a, P=P:
                            hf.aggregate_fuse_fwd(sh, c, self.agg, D, a["act"], a["Y"], a["R0"],
                                                  P["bias"], a["Z"], a["H"], a["fcnt"])))
                acts.append(a)
                X, gid = a["H"], None
                continue
            elif self.agg == "gat_xrel":     # softmax across relations (NEXT(2))
                ops.append((f"aggregate_fwd.{l}", lambda sh=sh, c=csrs[l], a=a:
                            hf.aggregate_fwd_xrel(sh, c, D, H, self.slope, a["Y"], a["s_src"],
                                                  a["s_dst"], a["Z"], a["stats"])))
            else:
                ops.append((f"aggregate_fwd.{l}", lambda sh=sh, c=csrs[l], a=a: hf.aggregate_fwd(
                    c, sh.rows, self.agg, D, H, self.slope, a["Y"], a["s_src"], a["s_dst"],
                    a["Z"], a["stats"])))
            if self.fusion == "han":
                a["beta"] = self._buf(f"beta{l}", max(sh.R, 1))
                a["wss"] = self._ws(hf.sem_att_ws_bytes(sh, D, D), key=f"ws_sem{l}")
                ops.append((f"fuse.{l}", lambda sh=sh, a=a, l=l: hf.semantic_fuse_att(
                    sh, D, D, a["act"], a["Z"], a["R0"], self.P[f"{l}.bias"],
                    self.P[f"{l}.sem_W"], self.P[f"{l}.sem_b"], self.P[f"{l}.sem_q"], a["beta"],
                    None, a["H"], a["wss"])))
            else:
                ops.append((f"fuse.{l}", lambda sh=sh, a=a, P=P: hf.semantic_fuse(
                    sh, D, a["act"], a["Z"], a["R0"], P["bias"], a["H"])))
            acts.append(a)
            X, gid = a["H"], None
        last = shapes[-1]
        dH = self._mat(f"dH{L - 1}", last.dst_rows, D)
        wsx = self._ws(hf.xent_ws_bytes(db.B, D, C), key="ws_xent")

        def side_op(fn):
            """Weight-gradient calls: on the side stream when split_head (a
            parallel graph branch, joined by the last op), else in line."""
            if not split_head:
                return fn

            def run():
                self._head_side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(self._head_side):
                    fn()
            return run

        Hl = acts[-1]["H"][:last.dst_rows]
        ops.append(("xent", lambda dH=dH: hf.linear_xent(
            db.B, D, C, Hl, db.h_row0, dev["labels"], self.P["Wc"], self.P["bc"], self.loss,
            dH[:last.dst_rows], None, None, wsx, status=self.status)))
        ops.append(("xent_wgrad", side_op(lambda: hf.linear_xent_wgrad(
            db.B, D, C, Hl, db.h_row0, self.Gd["Wc"], self.Gd["bc"], wsx))))
        if self.world > 1:
            ops.append(("allreduce.head", self._allreduce_op("head")))
        for l in range(L - 1, -1, -1):
            sh, a = shapes[l], acts[l]
            P = {k: self.P.get(f"{l}.{k}") for k in ("W_rel", "W_root", "bias", "att")}
            Gr = {k: self.Gd.get(f"{l}.{k}") for k in ("W_rel", "W_root", "bias", "att")}
            if self.agg_first and l == 0:
                b = dict(dH=dH, G=self._mat(f"G{l}", sh.dst_rows, D),
                         wsf=self._ws(hf.fuse_bwd_ws_bytes(sh, D)),
                         wsq=self._ws(hf.project_aggregated_bwd_ws_bytes(sh, a["K"], D)))
                self._fuse_bwd_ops(ops, l, sh, a, b, Gr, D, side_op)
                ops.append(("project_aggregated_bwd.0", lambda sh=sh, c=csrs[l], a=a, b=b, Gr=Gr:
                            hf.project_aggregated_bwd(sh, c, a["K"], D, a["Xagg"], a["Xroot"],
                                                      a["gid_root"], b["G"], Gr["W_rel"],
                                                      Gr["W_root"], b["wsq"], prec=self.prec_tc)))
                if self.world > 1:
                    ops.append((f"allreduce.{l}", self._allreduce_op(f"layer{l}")))
                continue
            b = dict(dH=dH, G=self._mat(f"G{l}", sh.dst_rows, D),
                     dY=self._mat(f"dY{l}", sh.U_max, D),
                     ds_src=self._mat(f"dss{l}", sh.U_max, H) if P["att"] is not None else None,
                     ds_dst=self._mat(f"dsd{l}", sh.rows, H) if P["att"] is not None else None,
                     dX=self._mat(f"dH{l - 1}", sh.src_rows, D) if l > 0 else None,
                     wsf=self._ws(hf.fuse_bwd_ws_bytes(sh, D)),
                     wsa=self._ws(hf.aggregate_bwd_ws_bytes(sh, self.agg, H)),
                     wsq=self._ws(hf.project_bwd_ws_bytes(sh, a["K"], D, H)))
            if self.fusion == "han":
                # HAN: per-merged-row gradient dZ, then the row-gradient adjoint
                b["dZ"] = self._mat(f"dZ{l}", sh.rows, D)
                ops.append((f"fuse_bwd.{l}", lambda sh=sh, a=a, b=b, l=l: hf.semantic_fuse_att_bwd(
                    sh, D, D, a["act"], b["dH"], a["H"], a["Z"], self.P[f"{l}.sem_W"],
                    self.P[f"{l}.sem_b"], self.P[f"{l}.sem_q"], a["beta"], b["G"], b["dZ"],
                    self.Gd[f"{l}.bias"], self.Gd[f"{l}.sem_W"], self.Gd[f"{l}.sem_b"],
                    self.Gd[f"{l}.sem_q"], a["wss"])))
                ops.append((f"aggregate_bwd.{l}", lambda sh=sh, c=csrs[l], a=a, b=b, P=P:
                            hf.aggregate_bwd_rows(sh, c, self.agg, D, H, self.slope, b["dZ"],
                                                  a["Y"], a["s_src"], a["s_dst"], a["stats"],
                                                  P["att"], b["dY"], b["ds_src"], b["ds_dst"],
                                                  b["wsa"])))
            else:
                self._fuse_bwd_ops(ops, l, sh, a, b, Gr, D, side_op)
            if self.fusion == "han":
                pass                   # aggregation adjoint queued above
            elif P["att"] is not None:   # RGAT: score chain folded into the CSC pass
                ops.append((f"aggregate_bwd.{l}", lambda sh=sh, c=csrs[l], a=a, b=b, P=P:
                            hf.aggregate_bwd_scored(sh, c, self.agg, D, H, self.slope, b["G"],
                                                    a["Y"], a["s_src"], a["s_dst"], a["stats"],
                                                    P["att"], b["dY"], b["ds_src"], b["ds_dst"],
                                                    b["wsa"])))
            else:
                ops.append((f"aggregate_bwd.{l}", lambda sh=sh, c=csrs[l], a=a, b=b:
                            hf.aggregate_bwd(sh, c, self.agg, D, H, self.slope, b["G"], a["Y"],
                                             a["s_src"], a["s_dst"], a["stats"], b["dY"],
                                             b["ds_src"], b["ds_dst"], b["wsa"])))
            if P["att"] is None and b["dX"] is not None:
                # RGCN inner layer: the input gradient (next on the critical
                # path) and the weight gradients as two calls, the second on
                # the side stream overlapping the outer layer's backward
                b["wsw"] = self._ws(hf.project_bwd_ws_bytes(sh, a["K"], D, H), key=f"ws_wg{l}")
                ops.append((f"project_bwd.{l}", lambda sh=sh, c=csrs[l], a=a, b=b, P=P:
                            hf.project_bwd(sh, c, a["K"], D, H, a["X"], a["gid"], P["W_rel"],
                                           P["W_root"], None, a["Y"], b["dY"], b["G"], None,
                                           None, b["dX"], None, None, None, b["wsq"],
                                           prec=self.prec_tc)))
                ops.append((f"project_wgrad.{l}", side_op(
                    lambda sh=sh, c=csrs[l], a=a, b=b, P=P, Gr=Gr:
                    hf.project_bwd(sh, c, a["K"], D, H, a["X"], a["gid"], P["W_rel"],
                                   P["W_root"], None, a["Y"], b["dY"], b["G"], None, None, None,
                                   Gr["W_rel"], Gr["W_root"], None, b["wsw"], prec=self.prec_tc))))
            elif P["att"] is not None and b["dX"] is not None:
                # RGAT inner layer: the input gradient (dgrad + the s_dst chain's
                # dX term) on the critical path, the weight / attention
                # gradients as a second call on the side stream, overlapping the
                # outer layer's backward (both calls read the dYt left by
                # hifuse_aggregate_bwd_scored / _rows)
                b["wsw"] = self._ws(hf.project_bwd_ws_bytes(sh, a["K"], D, H), key=f"ws_wg{l}")
                ops.append((f"project_bwd.{l}", lambda sh=sh, c=csrs[l], a=a, b=b, P=P:
                            hf.project_bwd_scored(sh, c, a["K"], D, H, a["X"], a["gid"],
                                                  P["W_rel"], P["W_root"], P["att"], a["Y"],
                                                  b["dY"], b["G"], b["ds_src"], b["ds_dst"],
                                                  b["dX"], None, None, None, b["wsq"],
                                                  prec=self.prec_tc)))
                ops.append((f"project_wgrad.{l}", side_op(
                    lambda sh=sh, c=csrs[l], a=a, b=b, P=P, Gr=Gr:
                    hf.project_bwd_scored(sh, c, a["K"], D, H, a["X"], a["gid"], P["W_rel"],
                                          P["W_root"], P["att"], a["Y"], b["dY"], b["G"],
                                          b["ds_src"], b["ds_dst"], None, Gr["W_rel"],
                                          Gr["W_root"], Gr["att"], b["wsw"],
                                          prec=self.prec_tc))))
            else:
                pb = hf.project_bwd_scored if P["att"] is not None else hf.project_bwd
                ops.append((f"project_bwd.{l}", lambda sh=sh, c=csrs[l], a=a, b=b, P=P, Gr=Gr,
                            pb=pb:
                            pb(sh, c, a["K"], D, H, a["X"], a["gid"], P["W_rel"], P["W_root"],
                               P["att"], a["Y"], b["dY"], b["G"], b["ds_src"], b["ds_dst"],
                               b["dX"], Gr["W_rel"], Gr["W_root"], Gr["att"], b["wsq"],
                               prec=self.prec_tc)))
            dH = b["dX"]
            if self.world > 1:
                ops.append((f"allreduce.{l}", self._allreduce_op(f"layer{l}")))
        if self.world > 1:
            ops.append(("allreduce_join", self._dp_join))
        if split_head:
            ops.append(("head_join", lambda: torch.cuda.current_stream().wait_stream(
                self._head_side)))
        self.last = dict(acts=acts, csrs=csrs)
        return ops

    def _fuse_bwd_ops(self, ops, l, sh, a, b, Gr, D, side_op):
        """Fusion backward: G = dH * act' on the critical path; the bias
        gradient (column sums of G, bit-identical to the combined call) as a
        weight-gradient op on the side stream."""
        ops.append((f"fuse_bwd.{l}", lambda sh=sh, a=a, b=b: hf.semantic_fuse_bwd(
            sh, D, a["act"], b["dH"], a["H"], b["G"], None, b["wsf"])))
        b["wsb"] = self._ws(hf.fuse_bwd_ws_bytes(sh, D), key=f"ws_fb{l}")
        ops.append((f"fuse_bwd_bias.{l}", side_op(lambda sh=sh, b=b, Gr=Gr:
                                                  hf.semantic_fuse_bwd_bias(sh, D, b["G"],
                                                                            Gr["bias"],
                                                                            b["wsb"]))))

    # ----------------------------------------------------------------- step
    def step(self, db: DeviceBatch, feat, edge_type, allreduce=None, world=1, update=True,
             prof=None):
        """Runs one training step eagerly on the current stream; returns the
        device loss tensor (no host synchronisation).  ``prof``: optional dict
        receiving (start, end) CUDA events around every library call."""
        def timed(name, fn):
            if prof is None:
                fn()
                return
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            prof.setdefault(name, []).append((a, b))

        for name, fn in self.plan(db, feat, edge_type):
            timed(name, fn)
        if allreduce is not None:
            timed("allreduce", lambda: allreduce(self.grads))
        if self.world > 1:
            world = self.world               # bucketed all-reduce ran inside the plan
        if update:
            timed("sgd", lambda: hf.sgd(self.params, self.grads, self.lr, 1.0 / world))
        return self.loss

    def capture(self, db: DeviceBatch, feat, edge_type, update=True, world=1):
        """CUDA graph of the whole step for batch ``db`` (compute + SGD when
        ``world == 1``; for world > 1 the SGD runs after the eager NCCL
        all-reduce).  Buffers must already have their final size (run one eager
        step per batch first).  Returns (graph, kernels launched per replay)."""
        ops = self.plan(db, feat, edge_type)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = hf.kernel_launches()
        with torch.cuda.graph(g, stream=self._cap):
            for _, fn in ops:
                fn()
            if update and (world == 1 or self.world > 1):
                # (bucketed in-graph all-reduce when set_dp was called: NCCL)
                hf.sgd(self.params, self.grads, self.lr, 1.0 / max(self.world, 1))
        return g, hf.kernel_launches() - n0

    def capture_pipelined(self, db: DeviceBatch, db_next: DeviceBatch, feat, edge_type, side,
                          update=True):
        """CUDA graph of one pipelined step: the semantic-graph build of the
        NEXT batch runs on stream ``side`` while batch ``db`` (built by the
        previous replay) goes through forward, backward and SGD on the
        capturing stream -- the B200 form of the paper's CPU/GPU pipeline
        (Fig. 6) with both sides on the GPU.
        Returns (graph, kernels launched per replay)."""
        ops = self.plan(db, feat, edge_type, include_build=False)
        bop = self.build_op(db_next, edge_type)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = hf.kernel_launches()
        # the compute chain is captured on a high-priority stream, the build on
        # the (default-priority) side stream: the block scheduler favours the
        # critical path and the latency-bound build fills the gaps
        with torch.cuda.graph(g, stream=self._hi):
            main = torch.cuda.current_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                bop()
            for _, fn in ops:
                fn()
            if update:
                hf.sgd(self.params, self.grads, self.lr, 1.0 / max(self.world, 1))
            main.wait_stream(side)
        return g, hf.kernel_launches() - n0

    def capture_stages(self, db: DeviceBatch, feat, edge_type):
        """One CUDA graph per library call of the step (for per-stage device
        timing); returns [(name, graph, kernels)]."""
        out = []
        ops = [(n, f) for n, f in self.plan(db, feat, edge_type, split_head=False)
               if not n.startswith("allreduce")]          # library calls only
        torch.cuda.synchronize()
        for name, fn in ops:
            g = torch.cuda.CUDAGraph()
            n0 = hf.kernel_launches()
            with torch.cuda.graph(g, stream=self._cap):
                fn()
            out.append((name, g, hf.kernel_launches() - n0))
        return out
