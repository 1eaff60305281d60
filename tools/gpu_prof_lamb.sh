cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
S=gpurun_out/status.txt
: > $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?" >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-parity --no-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu_launches=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:lamb_onchip" -s 3 -c 1 \
   -o gpurun_out/prof_lamb -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-parity --no-baseline > gpurun_out/ncu_lamb.log 2>&1; echo "ncu_lamb=$?" >> $S
