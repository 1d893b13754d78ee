# call y (session 3): hot tables retry with other multipliers before the two-way fallback
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py -q -x > gpurun_out/s3y_pytest.txt 2>&1; echo rc=$?
tail -3 gpurun_out/s3y_pytest.txt
timeout 900 python bench.py --config c3 --steps 6 --no-cpu-baseline --no-e2e > gpurun_out/s3y_bench_c3.json 2> gpurun_out/s3y_bench_c3.err; echo rc=$?
IG_HOT_IMPORTANT=1 timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/s3y_bench_c3_fallback.json 2>> gpurun_out/s3y_bench_c3.err; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c5 or c1" > gpurun_out/s3y_fullsize.txt 2>&1; echo rc=$?
tail -3 gpurun_out/s3y_fullsize.txt
timeout 900 python bench.py --config c5 --steps 4 --no-cpu-baseline --no-e2e > gpurun_out/s3y_bench_c5.json 2> gpurun_out/s3y_bench_c5.err; echo rc=$?
python - <<'P'
import json
for f in ['s3y_bench_c3','s3y_bench_c3_fallback','s3y_bench_c5']:
    try:
        j=json.load(open(f'gpurun_out/{f}.json'))
        print(f, round(j['value'],2), round(j['ms_per_step'],1), {k:round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'], j['gpu_launches'])
    except Exception as e: print(f, 'ERR', e)
P
