#!/bin/bash
# Finalize kernel: one bin per thread-group, slab groups split over PRNGD_FINALIZE_SPLIT threads
# (product 4; variants/lib_fs1.so = 1). Parity of the consumer tests, launch lists of a cfg5 bench
# run for both, alternating bench lines of the consume workloads.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "consume or stat or hist or peer or finalize or exact or wrap or mc" 2>&1 | tail -2
for lib in product fs1; do
  if [ $lib = product ]; then L=""; else L="PRNGD_LIB=$PWD/variants/lib_fs1.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/s2g_${lib}_cfg5_launches.csv \
      python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 > /dev/null 2>&1
  python - $lib <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(f"gpurun_out/s2g_{sys.argv[1]}_cfg5_launches.csv")) if len(r) > 10]
h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value"); m = h.index("Metric Name")
d = collections.defaultdict(list)
for r in rows[1:]:
    if r[m] == "gpu__time_duration.sum": d[r[k].split("(")[0][:60]].append(float(r[v].replace(",", "")))
for a, b in d.items():
    if "prngd" in a: print(sys.argv[1], len(b), a, "mean ns", round(sum(b) / len(b)))
PY
done
for i in 1 2; do
STEPS=50 TAG=split4 bash tools/quick_ab.sh cfg5:auto mrg26:auto:--consume
PRNGD_LIB=$PWD/variants/lib_fs1.so STEPS=50 TAG=split1 bash tools/quick_ab.sh cfg5:auto mrg26:auto:--consume
done
