# call w (session 3): two hot lookups in flight per group pair in the queued dense loop
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py -q -x > gpurun_out/s3w_pytest.txt 2>&1; echo rc=$?
tail -3 gpurun_out/s3w_pytest.txt
timeout 900 python bench.py --config c3 --steps 8 --no-cpu-baseline --no-e2e > gpurun_out/s3w_bench_c3.json 2> gpurun_out/s3w_bench_c3.err; echo rc=$?
grep "timed step" gpurun_out/s3w_bench_c3.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c5 or c1" > gpurun_out/s3w_fullsize.txt 2>&1; echo rc=$?
tail -3 gpurun_out/s3w_fullsize.txt
timeout 900 python bench.py --config c5 --no-cpu-baseline --no-e2e > gpurun_out/s3w_bench_c5.json 2> gpurun_out/s3w_bench_c5.err; echo rc=$?
grep "timed step" gpurun_out/s3w_bench_c5.err
python - <<'P'
import json
for f in ['s3w_bench_c3','s3w_bench_c5']:
    try:
        j=json.load(open(f'gpurun_out/{f}.json'))
        print(f, round(j['value'],2), round(j['ms_per_step'],1), {k:round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'], j['clocks']['samples'])
    except Exception as e: print(f, 'ERR', e)
P
