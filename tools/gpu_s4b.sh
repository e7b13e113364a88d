#!/bin/bash
# Session-4: where the fused consumer's shared-memory bank conflicts come from:
# per-op bank-conflict and wavefront counters of consume_kernel for cfg5 write + statistics
# (row segments, default), the ROW-tile layout, and statistics only (no tile at all).
mkdir -p gpurun_out
M='regex:l1tex__data_bank_conflicts_pipe_lsu_mem_shared.*sum$,regex:l1tex__data_pipe_lsu_wavefronts_mem_shared.*sum$,regex:smsp__inst_executed_op_shared.*sum$,regex:smsp__inst_executed_op_(ldsm|shared_atom|shared_red).*sum$,smsp__inst_executed.sum,gpu__time_duration.sum'
cap() { tag=$1; shift
  B="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 $*"
  $B > gpurun_out/s4b_${tag}_plain.log 2>&1 || { echo "plain $tag failed"; return; }
  timeout 600 ncu --metrics "$M" --clock-control none -k regex:consume_kernel -s 2 -c 1 --csv \
      --log-file gpurun_out/s4b_${tag}_smem.csv $B > /dev/null 2>&1
  echo "captured $tag rc=$?"; }
cap seg
cap row --store row
cap nowrite --no-write
echo done
