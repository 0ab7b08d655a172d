#!/bin/bash
# One GPU round: parity tests, C5 bench, C4@1e6 and C4@1e5 sketch benches (summary lines).
set -u
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
summ='import json,sys; d=json.loads(sys.stdin.read()); g=d.get("grad") or {}; print(d["config"]["workload"][:40], "step_ms=%.3f" % d["ms_per_step"], "sketch_ms=%.4f" % d["sketch"]["ms"], d["sketch"]["path"], "sk_frac=%.3f(%s)" % (d["sketch"]["roofline"]["frac"], d["sketch"]["roofline"]["bound"]), "grad_ms=%s" % g.get("ms_per_iter"), "grad_frac=%s" % (g.get("roofline") or {}).get("frac"), "cold=%s" % g.get("cold_l2_ms_per_launch"))'
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "$summ"
timeout 600 python bench.py --config C4 --n-per-pixel 1000000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4e6.log 2>&1; tail -1 gpurun_out/bench_c4e6.log | python -c "$summ"
timeout 300 python bench.py --config C4 --n-per-pixel 100000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4e5.log 2>&1; tail -1 gpurun_out/bench_c4e5.log | python -c "$summ"
