# call e: warp-queued cold probes + bucket probes; parity subset, c3 bench both ways, ncu
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_long_grams.py tests/test_gpu_configs.py -q -x -rf -m "not slow" > gpurun_out/pytest_new.txt 2>&1; echo rc_new=$?
tail -3 gpurun_out/pytest_new.txt
for env in "IG_HOT_SERIAL=1" "IG_HOT_Q=1"; do
  env $env timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$env.json 2> gpurun_out/bench_$env.err; echo rc=$?
  python -c "
import json; j=json.loads(open('gpurun_out/bench_$env.json').read().strip().splitlines()[-1]); print('$env', round(j['value'],2), round(j['ms_per_step'],1), j['result_digest'], {k: round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k})"
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/hot6q python bench.py --profile-run > gpurun_out/ncu_q.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/hot6q.ncu-rep --page details > gpurun_out/hot6q_details.txt 2>/dev/null
ncu -i gpurun_out/hot6q.ncu-rep --page source --csv > gpurun_out/hot6q_source.csv 2>/dev/null
rm -f gpurun_out/hot6q.ncu-rep
gzip -f gpurun_out/*_source.csv
timeout 900 python bench.py > gpurun_out/bench_c3_full.json 2> gpurun_out/bench_c3_full.err; echo rc_full=$?
tail -2 gpurun_out/bench_c3_full.err
