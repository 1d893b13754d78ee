# Quick perf iteration on the GPU box: parity subset + c2 device bench.
# usage: bash scripts/gpu_quick.sh [CONFIG]
CFG=${1:-c2}
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs.py -m "not slow" -x -q 2>&1 | tail -3
timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/quick_$CFG.json 2> gpurun_out/quick_$CFG.err
echo rc=$?
python - "$CFG" <<'PY'
import json, sys
j = json.load(open(f"gpurun_out/quick_{sys.argv[1]}.json"))
print("value", round(j["value"], 2), "ms", round(j["ms_per_step"], 2))
for k, v in j.get("kernel_breakdown", {}).items():
    print(f"  {k:14s} {v['ms_per_step']:8.2f} ms  x{v['launches_per_step']}")
print(" steps", {k: round(v, 2) for k, v in j.get("step_breakdown_ms", {}).items()})
PY
