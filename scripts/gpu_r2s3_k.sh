# call k (session 3): queued rank-bitmap 4-gram pass (IG_HOT_Q5) on the trimmed sweep
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IG_HOT_Q5=1 timeout 600 python -m pytest tests/test_gpu_count_all_paths.py -q -x > gpurun_out/s3k_pytest.txt 2>&1; echo rc=$?
tail -2 gpurun_out/s3k_pytest.txt
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export IG_HOT_Q5=1; else unset IG_HOT_Q5; fi
  timeout 900 python bench.py --config c3 --steps 6 --no-cpu-baseline --no-e2e > gpurun_out/s3k_bench_c3_q$v.json 2> gpurun_out/s3k_bench_c3.err; echo rc=$?
done
for v in 0 1; do
  if [ $v = 1 ]; then export IG_HOT_Q5=1; else unset IG_HOT_Q5; fi
  timeout 900 python bench.py --config c5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/s3k_bench_c5_q$v.json 2> gpurun_out/s3k_bench_c5.err; echo rc=$?
done
python - <<'P'
import json
for f in ['s3k_bench_c3_q0','s3k_bench_c3_q1','s3k_bench_c5_q0','s3k_bench_c5_q1']:
    try:
        j=json.load(open(f'gpurun_out/{f}.json'))
        print(f, round(j['value'],2), round(j['ms_per_step'],1), {k:round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'])
    except Exception as e: print(f, 'ERR', e)
P
