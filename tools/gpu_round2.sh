cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
S=gpurun_out/status.txt
: > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest=$?" >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gemm_pair" -s 3 -c 1 \
   -o gpurun_out/prof_gemm -f python tools/pattern_probe.py --only c3 --gemm-only > gpurun_out/ncu_gemm.log 2>&1; echo "ncu_gemm=$?" >> $S
