#!/bin/bash
# Finalize kernel, new (one bin per thread group, 4 slab groups) vs the round-2 version (32 blocks, serial chain per bin: variants/lib_fin_old.so).
# (product 4; variants/lib_fin_old.so = 1). Parity of the consumer tests, launch lists of a cfg5 bench
# run for both, alternating bench lines of the consume workloads.
mkdir -p gpurun_out
for lib in product fin_old; do
  if [ $lib = product ]; then L=""; else L="PRNGD_LIB=$PWD/variants/lib_fin_old.so"; fi
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
STEPS=50 TAG=new bash tools/quick_ab.sh cfg5:auto mrg26:auto:--consume cfg4:auto:--consume
PRNGD_LIB=$PWD/variants/lib_fin_old.so STEPS=50 TAG=old bash tools/quick_ab.sh cfg5:auto mrg26:auto:--consume cfg4:auto:--consume
done
