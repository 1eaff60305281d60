#!/bin/bash
# C1 through the reference-facing CLI flow on the GPU: goldens/adam.json +
# schedules/adam_fused.json at W=4, N=2^20 (the program as committed in
# tests/golden/adam_cases.json), EXACT and FAST, median device time of R runs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python - <<'PY'
import json
d = {c["name"]: c for c in json.load(open("tests/golden/adam_cases.json"))}
json.dump(d["adam_W4_N1048576"]["sched_program"], open("gpurun_out/c1_sched_program.json", "w"))
PY
for m in exact fast; do
  paper_2105_05720_b200/coconet-ccopt run gpurun_out/c1_sched_program.json --ranks 4 --size N=1048576 \
    --math $m --reps 20 | python -c "import json,sys; j=json.load(sys.stdin); print('$m', {k: j.get(k) for k in ('digest','deviation','device_ms','lowering')})"
done
