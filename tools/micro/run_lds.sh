#!/bin/bash
mkdir -p gpurun_out
./tools/micro/lds_bcast > gpurun_out/micro_lds.txt 2>&1 && \
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.per_second,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum --csv ./tools/micro/lds_bcast > gpurun_out/micro_lds_ncu.csv 2>&1
cat gpurun_out/micro_lds.txt
