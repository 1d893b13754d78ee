# hot-gram count-all: parity subset + c3 bench with kernel breakdown + slice/lgnb sweep
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_count_all_paths.py -x -q 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for env in "IG_NO_HOT=1" "" "IG_HOT_SLICE_MB=1000" "IG_HOT_SLICE_MB=100" "IG_HOT_SLICE_MB=24" "IG_HOT_LGNB=12"; do
  echo "== $env"
  env $env timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/hot_c3.json 2> gpurun_out/hot_c3.err || tail -5 gpurun_out/hot_c3.err
  python - <<'PY'
import json
j = json.load(open("gpurun_out/hot_c3.json"))
print("value", round(j["value"], 2), "ms", round(j["ms_per_step"], 2), "digest", j["result_digest"])
print(" steps", {k: round(v, 1) for k, v in j.get("step_breakdown_ms", {}).items()})
PY
done
