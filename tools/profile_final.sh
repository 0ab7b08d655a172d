#!/bin/bash
# End-of-round-2 captures at HEAD (tools only; one GPU): the bench launch list at C5 and
# `ncu --set full` of the hot kernels at C5, C1 and C4@1e2 (the configs the base-phasor V
# setup of sketch_tc.cu changes), summarised on the box into profiles/r02_final_*.json.
# Each command first runs without ncu (exit 0) as the profiling recipe requires.
set -u
O=gpurun_out
P=$O/r02f
mkdir -p $O $P
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-init --no-stream --no-sweep > $O/f_pre.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/f_launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-init --no-stream --no-sweep > $O/f_ncu_launch.log 2>&1
python tools/launch_summary.py $O/f_launches_c5.csv $P/r02_final_launches_c5.json > /dev/null
cp $O/f_launches_c5.csv $P/r02_final_launches_c5.csv
K='sketch_tc|grad_kernel'
for c in C5 C1; do
  python tools/prof_kernels.py $c --iters 1 > $O/f_pre_$c.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-count 4 \
      -o $O/f_$c python tools/prof_kernels.py $c --iters 1 > $O/f_ncu_$c.log 2>&1
  python tools/ncu_summary.py $O/f_$c.ncu-rep $P/r02_final_ncu_$c.json > /dev/null
  rm -f $O/f_$c.ncu-rep
done
python tools/prof_kernels.py C4 --n 100 --iters 0 > $O/f_pre_c4.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"sketch" --launch-count 1 -o $O/f_c4 \
    python tools/prof_kernels.py C4 --n 100 --iters 0 > $O/f_ncu_c4.log 2>&1
python tools/ncu_summary.py $O/f_c4.ncu-rep $P/r02_final_ncu_C4_100.json > /dev/null
rm -f $O/f_c4.ncu-rep
ls -la $P
