#!/bin/bash
# cfg2 in the bench context: kernel durations under ncu with the bench's own cache state
# (--cache-control none), new narrow kernel vs the previous one (variants/lib_jn0.so).
mkdir -p gpurun_out
for lib in product jn0; do
  if [ $lib = product ]; then L=""; else L="PRNGD_LIB=$PWD/variants/lib_jn0.so"; fi
  env $L ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none --cache-control none -k regex:gen_jump --csv \
     --log-file gpurun_out/s2d_${lib}_launches.csv python bench.py --workload cfg2 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 > /dev/null 2>&1
  python - "$lib" <<'PY'
import csv, sys, statistics
lib = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/s2d_{lib}_launches.csv")) if len(r) > 10]
hdr = rows[0]; iname = hdr.index("Metric Name"); ival = hdr.index("Metric Value"); ik = hdr.index("Kernel Name")
d = [float(r[ival].replace(",", "")) for r in rows[1:] if r[iname] == "gpu__time_duration.sum"]
c = [float(r[ival].replace(",", "")) for r in rows[1:] if r[iname] == "sm__cycles_active.avg"]
print(lib, rows[1][ik][:40], "n", len(d), "duration median", statistics.median(d), "min", min(d), "active cyc median", statistics.median(c))
PY
done
for i in 1 2 3; do
STEPS=300 TAG=new bash tools/quick_ab.sh cfg2:auto
PRNGD_LIB=$PWD/variants/lib_jn0.so STEPS=300 TAG=old bash tools/quick_ab.sh cfg2:auto
done
