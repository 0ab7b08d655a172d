#!/bin/bash
# ncu --set full (with SASS source) of the bucketing passes on a C5-sized stream (tools only).
set -u
O=gpurun_out
python tools/bucket_probe.py --time > $O/pre_bucket.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"partition_kernel|bucket_fine_kernel|coarse_count" \
    --launch-count 3 -o $O/bucket python tools/bucket_probe.py > $O/ncu_bucket.log 2>&1
python tools/ncu_summary.py $O/bucket.ncu-rep $O/bucket_sum.json > /dev/null
ncu -i $O/bucket.ncu-rep --page source --csv --print-source=sass -k regex:partition_kernel > $O/bucket_B_sass.csv
ncu -i $O/bucket.ncu-rep --page source --csv --print-source=sass -k regex:bucket_fine_kernel > $O/bucket_C_sass.csv
rm -f $O/bucket.ncu-rep
