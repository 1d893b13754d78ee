# call aa (session 3): sparse-tile walk threshold on c5 (IG_SPARSE_ITERS)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for it in 10 6 13 16; do
  IG_SPARSE_ITERS=$it timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s3aa_bench_c5_$it.json 2> gpurun_out/s3aa_bench_c5.err; echo rc=$?
done
python - <<'P'
import json
for it in [10,6,13,16]:
    try:
        j=json.load(open(f'gpurun_out/s3aa_bench_c5_{it}.json'))
        print(it, round(j['value'],2), round(j['ms_per_step'],1), {k:round(x,1) for k,x in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'])
    except Exception as e: print(it, 'ERR', e)
P
