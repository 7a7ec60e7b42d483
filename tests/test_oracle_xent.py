"""Pins of oracle.model.xent, the checker of the GPU classifier head
(hifuse_linear_xent / _wgrad): the linear classifier + mean softmax
cross-entropy that closes the step (reading C10).

Pinned against things other than its own formula: torch's fp64
cross_entropy + autograd (a library routine), closed forms (uniform logits:
loss = log C; two classes: the logistic loss), and central finite differences
of the loss for every gradient it returns."""
import math

import numpy as np
import pytest
import torch

import oracle.model as om


def _case(seed, B, D, C):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((B, D)), rng.standard_normal((D, C)) * 0.3,
            rng.standard_normal(C) * 0.1, rng.integers(0, C, B))


@pytest.mark.parametrize("B,D,C", [(7, 5, 3), (16, 8, 349), (33, 12, 2)])
def test_xent_matches_torch_autograd(B, D, C):
    hs, Wc, bc, lab = _case(B * C, B, D, C)
    ref = om.xent(hs, Wc, bc, lab)
    h = torch.tensor(hs, dtype=torch.float64, requires_grad=True)
    W = torch.tensor(Wc, dtype=torch.float64, requires_grad=True)
    b = torch.tensor(bc, dtype=torch.float64, requires_grad=True)
    loss = torch.nn.functional.cross_entropy(h @ W + b, torch.from_numpy(lab))
    loss.backward()
    assert abs(ref["loss"] - loss.item()) <= 1e-12 * max(1.0, abs(loss.item()))
    np.testing.assert_allclose(ref["dhs"], h.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(ref["dWc"], W.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(ref["dbc"], b.grad.numpy(), rtol=1e-10, atol=1e-14)


def test_xent_uniform_logits_closed_form():
    B, D, C = 9, 4, 5
    hs = np.random.default_rng(1).standard_normal((B, D))
    lab = np.arange(B) % C
    r = om.xent(hs, np.zeros((D, C)), np.zeros(C), lab)
    assert abs(r["loss"] - math.log(C)) < 1e-14
    want = np.full((B, C), 1.0 / C)
    want[np.arange(B), lab] -= 1.0
    np.testing.assert_allclose(r["dlog"], want / B, atol=1e-16)
    np.testing.assert_allclose(r["dhs"], 0.0, atol=1e-16)


def test_xent_two_classes_is_logistic_loss():
    B, D = 11, 3
    hs, Wc, bc, lab = _case(3, B, D, 2)
    r = om.xent(hs, Wc, bc, lab)
    z = hs @ Wc + bc
    margin = z[np.arange(B), lab] - z[np.arange(B), 1 - lab]
    want = np.mean(np.log1p(np.exp(-margin)))
    assert abs(r["loss"] - want) < 1e-13


def test_xent_finite_differences():
    B, D, C = 6, 4, 7
    hs, Wc, bc, lab = _case(5, B, D, C)
    r = om.xent(hs, Wc, bc, lab)
    h = 1e-6
    for name, arr, grad in (("hs", hs, r["dhs"]), ("Wc", Wc, r["dWc"]), ("bc", bc, r["dbc"])):
        for idx in np.ndindex(arr.shape):
            a1, a2 = arr.copy(), arr.copy()
            a1[idx] += h
            a2[idx] -= h
            args = {"hs": hs, "Wc": Wc, "bc": bc}
            f = []
            for a in (a1, a2):
                args[name] = a
                f.append(om.xent(args["hs"], args["Wc"], args["bc"], lab)["loss"])
            fd = (f[0] - f[1]) / (2 * h)
            assert abs(fd - grad[idx]) <= 1e-7 + 1e-5 * abs(grad[idx]), (name, idx, fd, grad[idx])
