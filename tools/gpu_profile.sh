#!/bin/bash
# Profiling session: pattern probe, bench, bench launch list, ncu full captures of
# the LAMB kernel (bench), the tcgen05 GEMM (C3 shape) and the PP boundary kernel (C4 fp16).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
S=gpurun_out/status.txt
: > $S
timeout 600 python tools/pattern_probe.py > gpurun_out/pattern_probe.log 2>&1; echo "pattern=$?" >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?" >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-parity --no-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu_launches=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${LAMB_KERNEL:-lamb_onchip}" -s 3 -c 1 \
   -o gpurun_out/prof_lamb -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-parity --no-baseline > gpurun_out/ncu_lamb.log 2>&1; echo "ncu_lamb=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gemm_pair" -s 3 -c 1 \
   -o gpurun_out/prof_gemm -f python tools/pattern_probe.py --only c3 --gemm-only > gpurun_out/ncu_gemm.log 2>&1; echo "ncu_gemm=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rs_send_ag" -s 8 -c 1 \
   -o gpurun_out/prof_pp -f python tools/pattern_probe.py --only c4 > gpurun_out/ncu_pp.log 2>&1; echo "ncu_pp=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:mp_ag_gemm" -s 3 -c 1 \
   -o gpurun_out/prof_ag -f python tools/pattern_probe.py --only c3 > gpurun_out/ncu_ag.log 2>&1; echo "ncu_ag=$?" >> $S
