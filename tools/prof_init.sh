#!/bin/bash
# ncu --set full of the tensor-core init_depths kernel at C5 (tools only): summary JSON, SASS source page.
set -u
O=gpurun_out
python tools/init_probe.py --config C5 --reps 2 ${PROF_ARGS:-} > $O/pre_init.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:bp_tc_kernel --launch-skip 3 --launch-count 1 \
    -o $O/init python tools/init_probe.py --config C5 --reps 2 ${PROF_ARGS:-} > $O/ncu_init.log 2>&1
python tools/ncu_summary.py $O/init.ncu-rep $O/init_sum.json > /dev/null
ncu -i $O/init.ncu-rep --page source --csv --print-source=sass > $O/init_sass.csv
rm -f $O/init.ncu-rep
