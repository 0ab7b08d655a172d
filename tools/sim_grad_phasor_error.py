"""Emulate the fp32 phasor chain of the expected-sketch / gradient kernels
(tools only): anchors from a 32-bit fixed-point phase q = round(frac(t/T) 2^32),
a = float(int32(j*q)) * 2^-31 half-revolutions, (cos, sin)(pi a) rounded to
fp32, then p_j = p_{j-1} * w between anchors (FMUL2+FFMA2 emulated).
Reports the worst |p_j - exp(i 2 pi j t / T)| over random real depths."""
import numpy as np

f32 = np.float32


def fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def anchor(q, j):
    s = ((q.astype(np.uint64) * np.uint64(j)) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    a = s.astype(np.float32) * f32(2.0 ** -31)
    return np.cos(np.pi * a.astype(np.float64)).astype(f32), np.sin(np.pi * a.astype(np.float64)).astype(f32)


def run(T, m, R, n=200000, seed=0):
    rng = np.random.default_rng(seed)
    t = rng.uniform(0, T, size=n).astype(np.float32)
    t[:20] = np.float32(T) - np.float32(2.0 ** -10) * np.arange(20)  # near the wrap
    q = np.floor(np.mod(t.astype(np.float64) / T, 1.0) * 2.0 ** 32 + 0.5).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    wc, ws = anchor(q, 1)
    pc, ps = wc, ws
    worst = 0.0
    for j in range(1, m + 1):
        if j > 1:
            if (j - 1) % R == 0:
                pc, ps = anchor(q, j)
            else:
                t1 = (pc.astype(np.float64) * wc).astype(f32)
                t2 = (pc.astype(np.float64) * ws).astype(f32)
                pc, ps = fma32(-ps, ws, t1), fma32(ps, wc, t2)
        ph = 2 * np.pi * np.mod(j * t.astype(np.float64), T) / T
        worst = max(worst, float(np.maximum(np.abs(pc - np.cos(ph)), np.abs(ps - np.sin(ph))).max()))
    return worst


if __name__ == "__main__":
    for T, m in [(1024, 4), (4613, 10), (2500, 20), (8192, 32), (65536, 64)]:
        print(T, m, {R: f"{run(T, m, R):.2e}" for R in (8, 16, 32, 64) if R <= max(m, 8)})
