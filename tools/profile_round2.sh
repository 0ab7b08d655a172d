#!/bin/bash
# Round-2 profile captures (tools only; one GPU): the bench launch list at
# C5 and one `ncu --set full` capture of every hot kernel at every BASELINE config (C1, C2,
# C3, C5, the C4 sweep), summarised on the box into profiles/r02_*.json (the .ncu-rep files
# are too large to bring back).  Each command first runs without ncu (exit 0) as the recipe
# requires.
set -u
O=gpurun_out
P=$O/r02
mkdir -p $O $P
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-init --no-stream --no-sweep > $O/pre.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-init --no-stream --no-sweep > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches_c5.csv $P/r02_launches_c5.json > /dev/null
K='sketch_kernel|sketch_routed|sketch_tc|sketch_hist|grad_kernel|fit_kernel|bp_tc_kernel|backproject_kernel|init_k1|merge_kernel'
for c in C5 C3 C2 C1; do
  python tools/prof_kernels.py $c --iters 1 --next > $O/pre_$c.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip 0 --launch-count 12 \
      -o $O/$c python tools/prof_kernels.py $c --iters 1 --next > $O/ncu_$c.log 2>&1
  python tools/ncu_summary.py $O/$c.ncu-rep $P/r02_ncu_$c.json > /dev/null
  rm -f $O/$c.ncu-rep
done
for n in 100 1000 10000 100000 1000000; do
  python tools/prof_kernels.py C4 --n $n --iters 0 > $O/pre_c4_$n.log 2>&1 || exit 1
  ncu --set full --clock-control none -k regex:"sketch" --launch-count 1 -o $O/c4_$n \
      python tools/prof_kernels.py C4 --n $n --iters 0 > $O/ncu_c4_$n.log 2>&1
  python tools/ncu_summary.py $O/c4_$n.ncu-rep $P/r02_ncu_C4_$n.json > /dev/null
  rm -f $O/c4_$n.ncu-rep
done
python tools/bucket_probe.py > $O/pre_bk.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"coarse_count|partition_kernel|bucket_fine" --launch-count 3 \
    -o $O/bucket python tools/bucket_probe.py > $O/ncu_bk.log 2>&1
python tools/ncu_summary.py $O/bucket.ncu-rep $P/r02_ncu_bucket.json > /dev/null
rm -f $O/bucket.ncu-rep
ls -la $P/r02_*
