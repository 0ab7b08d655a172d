#!/bin/bash
# ncu --set full of the tensor-core sketch at C5 (tools only): summary JSON, raw CSV, SASS source page.
set -u
O=gpurun_out
python tools/prof_sketch.py --path 5 --reps 1 ${PROF_ARGS:-} > $O/pre_tc.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sketch_tc --launch-skip 1 --launch-count 1 \
    -o $O/tc python tools/prof_sketch.py --path 5 --reps 1 ${PROF_ARGS:-} > $O/ncu_tc.log 2>&1
python tools/ncu_summary.py $O/tc.ncu-rep $O/tc_sum.json > /dev/null
ncu -i $O/tc.ncu-rep --page raw --csv > $O/tc_raw.csv
ncu -i $O/tc.ncu-rep --page source --csv --print-source=sass > $O/tc_sass.csv
rm -f $O/tc.ncu-rep
