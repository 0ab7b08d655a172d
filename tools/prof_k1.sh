O=gpurun_out
python tools/init_probe.py --config C5 --reps 2 > $O/pre_k1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:init_k1 --launch-skip 2 --launch-count 2 -o $O/k1 python tools/init_probe.py --config C5 --reps 2 > $O/ncu_k1.log 2>&1
python tools/ncu_summary.py $O/k1.ncu-rep $O/k1_sum.json > /dev/null
ncu -i $O/k1.ncu-rep --page source --csv --print-source=sass > $O/k1_sass.csv
rm -f $O/k1.ncu-rep
