"""Per-config results table for BASELINE.md §4 (tools only; run on the GPU box):
bench.py for every BASELINE config (C4 at each sweep point) with the oracle
baseline, one markdown row per (config, kernel)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = [("C1", None), ("C2", None), ("C3", None), ("C5", None)] + [("C4", n) for n in (100, 1000, 10000, 100000, 1000000)]


def run(cfg, n):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "5", "--warmup", "3",
           "--no-e2e", "--no-init", "--no-stream", "--no-sweep", "--cpu-seconds", "6"]  # (fit: timed by default)
    if n:
        cmd += ["--n-per-pixel", str(n)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def main():
    rows = ["| Config | Kernel | GPU time | photons/s or px-it/s | GB/s (alg.) | % of roofline (bound) | SM clock | "
            "Oracle all-core | Oracle 1-core | Parity |", "|---|---|---|---|---|---|---|---|---|---|"]
    for cfg, n in RUNS:
        d = run(cfg, n)
        name = f"{cfg}@{n:.0e}".replace("+0", "") if n else cfg
        sk, g, cpu = d["sketch"], d.get("grad"), d.get("cpu_baseline") or {}
        clk = d.get("clocks", {}).get("sm_mhz")
        one = (cpu.get("one_core") or {}).get("value")
        rf = sk["roofline"]
        rows.append(f"| {name} | sketch ({sk['path']}) | {sk['ms']:.4f} ms | {sk['photons_per_s']:.3g} photons/s | "
                    f"{sk['gbs']:.0f} | {100 * rf['frac']:.1f} % ({rf['bound']}) | {clk} MHz | "
                    f"{cpu.get('value', 0):.3g} photons/s ({cpu.get('cores')} cores) | "
                    f"{one:.3g} photons/s | ≤1e-5 (tests) |" if one else
                    f"| {name} | sketch ({sk['path']}) | {sk['ms']:.4f} ms | {sk['photons_per_s']:.3g} photons/s | "
                    f"{sk['gbs']:.0f} | {100 * rf['frac']:.1f} % ({rf['bound']}) | {clk} MHz | – | – | ≤1e-5 (tests) |")
        if g:
            gr, gc = g["roofline_in_loop"], g["roofline"]
            rows.append(f"| {name} | gradient step (in loop; L2-cold launch) | {1000 * g['ms_per_iter']:.2f} µs/iter; "
                        f"{1000 * g['cold_l2_ms_per_launch']:.2f} µs | "
                        f"{g['pixel_iters_per_s']:.3g} px-it/s | {g['gbs']:.0f} | {100 * gr['frac']:.1f} %; cold "
                        f"{100 * gc['frac']:.1f} % ({gr['bound']}) | {clk} MHz | "
                        f"(step, above) | | A12 (tests) |")
        ft = d.get("fit")
        if ft:
            fr = ft["roofline"]
            rows.append(f"| {name} | fused fit ({ft['iters']} iterations, one launch) | {ft['ms']:.4f} ms | "
                        f"{ft['pixel_iters_per_s']:.3g} px-it/s | – | {100 * fr['frac']:.1f} % ({fr['bound']}) | "
                        f"{clk} MHz | | | bitwise = steps (tests) |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
