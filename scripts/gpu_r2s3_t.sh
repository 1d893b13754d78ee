# call t (session 3): what a very hot gram costs when it is NOT in the hot table
# (IG_HOT_DROP_ABOVE=c leaves grams with a sample count above c to the L2 REDs;
# the c3 sample is 67 M positions: c = 300000 / 60000 / 6000 is f > 0.45 % / 0.09 % / 0.009 %)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in none 300000 60000 6000; do
  if [ $c = none ]; then unset IG_HOT_DROP_ABOVE; else export IG_HOT_DROP_ABOVE=$c; fi
  timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s3t_bench_c3_$c.json 2> gpurun_out/s3t_bench_c3.err; echo rc=$?
done
python - <<'P'
import json
for c in ['none','300000','60000','6000']:
    try:
        j=json.load(open(f'gpurun_out/s3t_bench_c3_{c}.json'))
        print(c, round(j['value'],2), round(j['ms_per_step'],1), {k:round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'])
    except Exception as e: print(c, 'ERR', e)
P
