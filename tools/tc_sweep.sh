for c in C1 C2 C3 C5; do timeout 300 python tools/sketch_path_probe.py --config $c --only tensor --reps 10 2>&1 | tail -1; done
for n in 100 1000 10000 100000; do timeout 300 python tools/sketch_path_probe.py --config C4 --n $n --only tensor --reps 10 2>&1 | tail -1; done
