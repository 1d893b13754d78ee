# call b (session 3): mask-gated corpus loads, queued rank-bitmap pass (IG_HOT_Q5), c3 step gaps
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s3b_bench_c3_1.json 2> gpurun_out/s3b_bench_c3.err; echo rc=$?
timeout 900 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s3b_bench_c3_2.json 2>> gpurun_out/s3b_bench_c3.err; echo rc=$?
IG_HOT_Q5=1 timeout 900 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s3b_bench_c3_q5.json 2>> gpurun_out/s3b_bench_c3.err; echo rc=$?
grep "timed step" gpurun_out/s3b_bench_c3.err
timeout 1500 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py -q -x > gpurun_out/s3b_pytest.txt 2>&1; echo rc=$?
tail -3 gpurun_out/s3b_pytest.txt
timeout 900 python bench.py --config c5 --no-cpu-baseline --no-e2e > gpurun_out/s3b_bench_c5.json 2> gpurun_out/s3b_bench_c5.err; echo rc=$?
IG_HOT_Q5=1 timeout 900 python bench.py --config c5 --no-cpu-baseline --no-e2e > gpurun_out/s3b_bench_c5_q5.json 2>> gpurun_out/s3b_bench_c5.err; echo rc=$?
grep "timed step" gpurun_out/s3b_bench_c5.err
python - <<'P'
import json
for f in ['s3b_bench_c3_1','s3b_bench_c3_2','s3b_bench_c3_q5','s3b_bench_c5','s3b_bench_c5_q5']:
    try:
        j=json.load(open(f'gpurun_out/{f}.json'))
        print(f, round(j['value'],2), round(j['ms_per_step'],1), {k:round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'], j['clocks']['samples'])
    except Exception as e: print(f, 'ERR', e)
P
