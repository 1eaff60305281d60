#!/bin/bash
# One gpurun session: smoke, GPU tests, probe, bench, ncu launch list + one full capture.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
S=gpurun_out/status.txt
: > $S
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1; echo "pytest=$?" >> $S
if [ -n "$PROBE" ]; then timeout 600 python tools/probe.py > gpurun_out/probe.log 2>&1; echo "probe=$?" >> $S; fi
if [ -n "$BENCH" ]; then timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?" >> $S; fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu_launches=$?" >> $S
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNEL:-lamb}" -s 3 -c 1 \
     -o gpurun_out/prof_${NCU_KERNEL:-lamb} -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?" >> $S
fi
