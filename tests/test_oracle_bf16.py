"""Pins of oracle.bf16_round (reading C24, the BF16 projection's operand
rounding): hand-worked ties and ulps of the bfloat16 format (8 significand
bits), agreement with an independent library routine (torch's float ->
bfloat16 conversion, round-to-nearest-even), and invariants."""
import numpy as np
import torch

import oracle


def test_bf16_round_worked_values():
    ulp = 2.0 ** -7                      # bfloat16 ulp at [1, 2)
    cases = [
        (1.0, 1.0),
        (1.0 + ulp, 1.0 + ulp),          # representable
        (1.0 + ulp / 2, 1.0),            # tie -> even (1.0 has lowest bit 0)
        (1.0 + 3 * ulp / 2, 1.0 + 2 * ulp),   # tie -> even (up)
        (1.0 + ulp / 2 + 2.0 ** -20, 1.0 + ulp),   # just above the tie -> up
        (1.0 + ulp / 2 - 2.0 ** -20, 1.0),         # just below -> down
        (-3.0 - 3 * 2.0 ** -7, -3.0 - 4 * 2.0 ** -7),   # ulp 2^-6 at [2, 4): tie -> even
        (0.0, 0.0),
        (65280.0, 65280.0),              # 0x477F00: 255 * 256
        (2.0 ** -130, 2.0 ** -130),      # fp32 subnormal, representable (few bits)
    ]
    for x, want in cases:
        got = float(oracle.bf16_round(np.float32(x)))
        assert got == want, (x, got, want)


def test_bf16_round_matches_library_conversion():
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-6, 6, 20000),
                        rng.integers(-2 ** 12, 2 ** 12, 4000) / 64.0]).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(oracle.bf16_round(x), want)


def test_bf16_round_invariants():
    rng = np.random.default_rng(6)
    x = rng.standard_normal(5000).astype(np.float32)
    r = oracle.bf16_round(x)
    np.testing.assert_array_equal(oracle.bf16_round(r), r)              # idempotent
    np.testing.assert_array_equal(oracle.bf16_round(-x), -r)            # odd
    assert (np.abs(r - x) <= np.abs(x) * 2.0 ** -8 + 1e-45).all()      # half an ulp
    assert (r.astype(np.float32).view(np.uint32) & 0xFFFF == 0).all()   # 16 low bits clear
