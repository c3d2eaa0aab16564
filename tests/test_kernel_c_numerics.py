"""CPU checks of two numerical claims kernel (c) rests on (Q28, Q29).
They pin the arithmetic rules, evaluated here in numpy float32 exactly as the
CUDA code states them; the GPU parity suites check the kernels themselves.

Q28: a per-axis origin c = fl32((lo + hi) / 2) accepted by the rule
     c/2 <= lo and hi <= 2c (mirrored for negative boxes) makes x - c exact
     in FP32 for every float x in [lo, hi] (Sterbenz's lemma).
Q29: the degree-5 2^f fit of ex2_poly2 (coefficients read from k_repulse.cu)
     with the 1.5 * 2^23 rounding shifter and the exponent-field add gives 2^y
     to <= 3e-7 relative over the clamp range [-125, 126]."""
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
f32 = np.float32


def frame_origin(lo: float, hi: float) -> float:
    lo, hi = f32(lo), f32(hi)
    m = f32(f32(0.5) * lo + f32(0.5) * hi)
    ok = (lo > 0 and f32(0.5) * m <= lo and hi <= f32(2.0) * m) or \
         (hi < 0 and f32(0.5) * m >= hi and lo >= f32(2.0) * m)
    return float(m) if ok else 0.0


def test_frame_origin_subtraction_is_exact():
    rng = np.random.default_rng(3)
    accepted = 0
    for _ in range(400):
        centre = rng.choice([-1.0, 1.0]) * 10.0 ** rng.uniform(-3, 6)
        half = abs(centre) * 10.0 ** rng.uniform(-6, 0.3)
        lo, hi = f32(centre - half), f32(centre + half)
        c = frame_origin(lo, hi)
        if c == 0.0:
            continue
        accepted += 1
        x = rng.uniform(float(lo), float(hi), size=2000).astype(np.float32)
        x = np.concatenate([x, [lo, hi]]).astype(np.float32)
        d32 = (x - f32(c)).astype(np.float64)
        d64 = x.astype(np.float64) - float(c)
        assert np.array_equal(d32, d64), (lo, hi, c)
    assert accepted > 100


def test_frame_origin_rejects_boxes_reaching_zero():
    assert frame_origin(-1.0, 5.0) == 0.0
    assert frame_origin(0.0, 5.0) == 0.0
    assert frame_origin(1.0, 10.0) == 0.0      # spans a factor > 3
    assert frame_origin(885.0, 1140.0) != 0.0  # cfg4's layout (profiles/README.md)
    assert frame_origin(-1140.0, -885.0) != 0.0


def _poly_coefficients():
    src = open(os.path.join(ROOT, "paper_1506_04383_b200", "csrc", "k_repulse.cu")).read()
    body = src[src.index("ex2_poly2(f2x y)"):]
    body = body[:body.index("upk(p, p0, p1)")]
    first = re.search(r"f2x p = pk\(([-0-9.e]+)f", body).group(1)
    rest = re.findall(r"p = fma2\(p, f, pk\(([-0-9.e]+)f", body)
    return [f32(first)] + [f32(c) for c in rest]  # highest degree first


def ex2_poly(y: np.ndarray) -> np.ndarray:
    shift = f32(12582912.0)
    y = np.minimum(np.maximum(y.astype(np.float32), f32(-125.0)), f32(126.0))
    t = (y + shift).astype(np.float32)
    tm = (t - shift).astype(np.float32)
    fr = (y - tm).astype(np.float32)
    c = _poly_coefficients()
    p = np.full_like(fr, c[0])
    for a in c[1:]:
        p = (p * fr + a).astype(np.float32)  # FFMA rounding differs by <= 1 ulp from this
    n = t.view(np.int32) - np.int32(0x4B400000)
    return (p.view(np.int32) + (n << 23)).view(np.float32)


def test_ex2_poly_accuracy():
    c = _poly_coefficients()
    assert len(c) == 6
    y = np.concatenate([np.linspace(-125.0, 126.0, 400001), np.arange(-125, 126) + 0.5]).astype(np.float32)
    got = ex2_poly(y).astype(np.float64)
    want = np.exp2(y.astype(np.float64))
    # outside the range the clamp applies (as in inv_pow's kExpClamp for the MUFU path)
    assert ex2_poly(np.array([200.0], np.float32))[0] == ex2_poly(np.array([126.0], np.float32))[0]
    rel = np.abs(got / want - 1.0)
    assert rel.max() <= 3e-7, rel.max()
