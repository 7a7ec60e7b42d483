"""Helpers shared by the -m gpu parity tests (CUDA path vs the CPU oracle)."""
import numpy as np
import pytest
import torch

import oracle

needs_gpu = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
DEV = "cuda:0"


def hf():
    import paper_2408_08490_b200.hifuse as h
    return h


def gpu_build(blk, et, rel_src, rel_dst, status=None, csc=True, ranged=False, xrow=False,
              x_gather=None):
    """Runs hifuse_build_semantic_graphs on one layer; returns (shape, csr).
    ranged: pass the relation-major offsets of `et` instead of the table."""
    h = hf()
    sh = h.Shape(rel_src, rel_dst, blk.n_src, blk.n_dst, blk.num_edges)
    csr = h.CsrBuffers(sh, DEV, csc=csc, xrow=xrow)
    if x_gather is not None:
        csr.set_x_gather(x_gather)
    ws = torch.empty((sh.build_ws + 3) // 4 + 16, dtype=torch.int32, device=DEV)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=DEV)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(DEV)
    et_d = t(et, np.int32)
    off = None
    if ranged:
        off = torch.empty(sh.R + 1, dtype=torch.int64, device=DEV)
        st2 = torch.zeros(1, dtype=torch.int32, device=DEV)
        h.edge_type_offsets(et_d, sh.R, off, st2)
        assert h.read_status(st2) == 0, "edge types not relation-major"
    h.build_semantic_graphs([sh], [csr], [t(blk.src_local, np.int32)], [t(blk.dst_local, np.int32)],
                            [t(blk.edge_id, np.int64)], et_d, ws, st, rel_edge_off=off)
    torch.cuda.synchronize()
    return sh, csr, st


def csr_host(sh, csr):
    U = int(csr["U_dev"].item())
    g = lambda k, n: None if csr[k] is None else csr[k][:n].cpu().numpy()
    return dict(U=U, rel_row_off=g("rel_row_off", sh.R + 1), row_ptr=g("row_ptr", sh.rows + 1),
                col=g("col", sh.N), eperm=g("eperm", sh.N), rel_y_off=g("rel_y_off", sh.R + 1),
                y_src=g("y_src", U), col_ptr=g("col_ptr", U + 1), csc_pos=g("csc_pos", sh.N),
                csc_row=g("csc_row", sh.N), csc_col=g("csc_col", sh.N), slot_y=g("slot_y", sh.S))


def assert_build_equal(gpu, ref):
    assert gpu["U"] == ref["U"]
    for k in ("rel_row_off", "row_ptr", "col", "eperm", "rel_y_off", "y_src", "col_ptr",
              "csc_pos", "csc_row", "csc_col", "slot_y"):
        assert np.array_equal(gpu[k], np.asarray(ref[k])), k


def close_scaled(g, r, scale, rtol=1e-5, what=""):
    """|g - r| <= rtol * max(|r|, scale) per element."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    bound = rtol * np.maximum(np.abs(r), np.asarray(scale, np.float64)) + 1e-30
    err = np.abs(g - r)
    bad = err > bound
    assert not bad.any(), (f"{what}: {bad.sum()} of {bad.size} elements out of tolerance; "
                           f"worst err {err.max():.3e} (rel {np.max(err / bound) * rtol:.3e})")


def row_rel_l2(g, r, tol, what=""):
    """||g_i - r_i||_2 <= tol ||r_i||_2 per row (projection tolerance)."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    num = np.linalg.norm(g - r, axis=1)
    den = np.linalg.norm(r, axis=1)
    bad = num > tol * den + 1e-30
    assert not bad.any(), f"{what}: {bad.sum()} rows exceed {tol}; worst {np.max(num / (den + 1e-30)):.3e}"


def t(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)
