for r in 1 2; do
for v in default trig; do
  L=""; [ $v = trig ] && L="--lib tools/libsrt3d_trig.so"
  echo "== $v run $r"; timeout 200 python tools/grad_probe.py $L 2>&1 | tail -3
done; done
cp paper_2203_00952_b200/libsrt3d.so /tmp/libsave.so
for v in default trig default trig; do
  [ $v = trig ] && cp tools/libsrt3d_trig.so paper_2203_00952_b200/libsrt3d.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-init --no-stream --no-sweep > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['grad']; print('$v', d['ms_per_step'], g.get('ms_per_iter'), g.get('cold_l2_ms_per_launch'))"
  cp /tmp/libsave.so paper_2203_00952_b200/libsrt3d.so
done
