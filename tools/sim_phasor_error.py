"""Emulate the fp32 phasor recurrences of the sketch kernel (tools only).

For every photon bin x in [0, T) it runs the packed complex-power recurrence
p_j = p_{j-1} * w (FMUL2 + FFMA2, re-anchored from the exact-index table
every R terms) in emulated fp32 (products exact in fp64, then rounded), and
reports the worst |p_j - exp(i 2 pi j x / T)| over all x and j <= m.
Used to choose R (DESIGN.md §5 "phasor accuracy")."""
import sys
import numpy as np

f32 = np.float32


def fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def run(T, m, R):
    x = np.arange(T, dtype=np.int64)
    r = np.arange(T, dtype=np.float64)
    tab_c = np.cos(2 * np.pi * r / T).astype(f32)
    tab_s = np.sin(2 * np.pi * r / T).astype(f32)
    wc, ws = tab_c[x], tab_s[x]
    pc, ps = wc.copy(), ws.copy()
    worst = 0.0
    for j in range(1, m + 1):
        if j > 1:
            if (j - 1) % R == 0:
                idx = (j * x) % T
                pc, ps = tab_c[idx], tab_s[idx]
            else:
                # re' = fma(-ps, ws, pc*wc) ; im' = fma(ps, wc, pc*ws)
                t1 = (pc.astype(np.float64) * wc).astype(f32)
                t2 = (pc.astype(np.float64) * ws).astype(f32)
                nc = fma32(-ps, ws, t1)
                ns = fma32(ps, wc, t2)
                pc, ps = nc, ns
        ex = np.exp(2j * np.pi * ((j * x) % T) / T)
        err = np.abs(pc.astype(np.float64) - ex.real) + 0 * 1j
        err = np.maximum(np.abs(pc - ex.real), np.abs(ps - ex.imag))
        worst = max(worst, float(err.max()))
    return worst


if __name__ == "__main__":
    for T, m in [(1024, 4), (4613, 10), (2500, 20), (4096, 10), (8192, 32), (65536, 64)]:
        print(T, m, {R: f"{run(T, m, R):.2e}" for R in (8, 16, 32, 64) if R <= max(m, 8)})
