#!/bin/bash
# Round profile captures (tools only; one GPU): the bench launch list at C5 and
# one `ncu --set full` capture per hot kernel.  Each command first runs without
# ncu (exit 0) as the recipe requires.
set -u
O=gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-init --no-stream > $O/pre.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-init --no-stream > $O/ncu_launch.log 2>&1
python tools/prof_kernels.py C5 --iters 3 --next > $O/pre2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"sketch_kernel|grad_kernel|fit_kernel|backproject|bp_tc_kernel|init_k1|merge_kernel" \
    --launch-skip 0 --launch-count 10 -o $O/c5_full python tools/prof_kernels.py C5 --iters 1 --next > $O/ncu_c5.log 2>&1
python tools/prof_kernels.py C4 --n 1000000 --iters 0 > $O/pre3.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:sketch_hist --launch-count 1 -o $O/c4e6_hist python tools/prof_kernels.py C4 --n 1000000 --iters 0 > $O/ncu_c4.log 2>&1
ncu --set full --clock-control none -k regex:sketch_hist --launch-count 1 -o $O/c3_hist python tools/prof_kernels.py C3 --iters 0 > $O/ncu_c3.log 2>&1
ncu --set full --clock-control none -k regex:"coarse_count|partition_kernel|bucket_fine" --launch-count 3 -o $O/bucket_full python tools/bucket_probe.py > $O/ncu_bk.log 2>&1
ls $O/*.ncu-rep
# summaries (the .ncu-rep files are too large to bring back together)
python tools/launch_summary.py $O/launches_c5.csv $O/r01_launches_c5.json > /dev/null
for r in c5_full c4e6_hist c3_hist bucket_full; do
  python tools/ncu_summary.py $O/$r.ncu-rep $O/r01_ncu_$r.json > /dev/null
done
rm -f $O/*.ncu-rep
