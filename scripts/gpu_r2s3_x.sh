# call x (session 3): queue-less branch-free packed-set pass (IG_HOT_BF3) vs the queued sweep
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export IG_HOT_BF3=1; else unset IG_HOT_BF3; fi
  timeout 900 python bench.py --config c3 --steps 4 --no-cpu-baseline --no-e2e > gpurun_out/s3x_bench_c3_$v.json 2> gpurun_out/s3x_bench_c3.err; echo rc=$?
done
python - <<'P'
import json
for v in [0,1]:
    try:
        j=json.load(open(f'gpurun_out/s3x_bench_c3_{v}.json'))
        print(v, round(j['value'],2), round(j['ms_per_step'],1), {k:round(x,1) for k,x in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'])
    except Exception as e: print(v, 'ERR', e)
P
