#!/bin/bash
# Sketch / gradient summary for every BASELINE config (tools only; one GPU).
summ='import json,sys; d=json.loads(sys.stdin.read()); g=d.get("grad") or {}; s=d["sketch"]; print(d["config"]["workload"][:28], "| sketch %.4f ms %s G=%s frac=%.3f(%s)" % (s["ms"], s["path"], s["lanes_per_pixel"], s["roofline"]["frac"], s["roofline"]["bound"]), "| grad/iter", g.get("ms_per_iter"), "frac", (g.get("roofline") or {}).get("frac"))'
for c in C1 C2 C3 C5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-init --no-stream 2>/dev/null | tail -1 | python -c "$summ"
done
for n in 100 1000 10000 100000 1000000; do
  timeout 300 python bench.py --config C4 --n-per-pixel $n --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-init --no-stream 2>/dev/null | tail -1 | python -c "$summ"
done
