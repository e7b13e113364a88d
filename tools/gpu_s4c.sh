#!/bin/bash
# Session-4: shared-memory wavefronts of the tile patterns in isolation (tools/probe/lds_pattern.cu).
mkdir -p gpurun_out
./tools/probe/lds_pattern > gpurun_out/s4c_lds_plain.log 2>&1 || { echo plain failed; cat gpurun_out/s4c_lds_plain.log; exit 1; }
M='l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum'
timeout 600 ncu --metrics "$M" --clock-control none --csv --log-file gpurun_out/s4c_lds_smem.csv ./tools/probe/lds_pattern > /dev/null 2>&1
echo "ncu rc=$?"
