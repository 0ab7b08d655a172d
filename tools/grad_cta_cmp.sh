#!/bin/bash
# compare gradient-kernel CTA sizes (library variants) on the C5 bench
for v in default b8 b12; do
  if [ $v != default ]; then cp paper_2203_00952_b200/libsrt3d.so /tmp/libsave.so; cp tools/libsrt3d_$v.so paper_2203_00952_b200/libsrt3d.so; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.log 2>&1
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['grad']; print('$v', d['ms_per_step'], g['ms_per_iter'], g['cold_l2_ms_per_launch'])"
  if [ $v != default ]; then cp /tmp/libsave.so paper_2203_00952_b200/libsrt3d.so; fi
done
