cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
S=gpurun_out/status.txt
: > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest=$?" >> $S
# compute-sanitizer is closed on this pool; run it where it is allowed:
[ -n "$COCONET_SANITIZE" ] && for t in memcheck racecheck synccheck; do timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_$t.log 2>&1; echo "san_$t=$?" >> $S; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?" >> $S
