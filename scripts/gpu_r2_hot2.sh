cd /root/repo
timeout 900 python -m pytest tests/test_gpu_count_all_paths.py -x -q 2>&1 | tail -2
for env in "" "IG_HOT_SLICES=2" "IG_HOT_LGNB=12"; do
  echo "== $env"
  env $env timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/hot_c3.json 2> gpurun_out/hot_c3.err || tail -5 gpurun_out/hot_c3.err
  python - <<'PY'
import json
j = json.load(open("gpurun_out/hot_c3.json"))
print("value", round(j["value"], 2), "ms", round(j["ms_per_step"], 2), "digest", j["result_digest"])
print(" steps", {k: round(v, 1) for k, v in j.get("step_breakdown_ms", {}).items()})
PY
done
python bench.py --config c3 --profile-run > gpurun_out/plain_c3h.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_hot -c 11 -o gpurun_out/r13_c3_hot python bench.py --config c3 --profile-run > gpurun_out/ncu_c3h.log 2>&1
echo rc_ncu=$?; tail -3 gpurun_out/ncu_c3h.log
