# call s (session 3): hot-set sample stride 64 / 128 / 256 on c3
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for st in 64 128 256 32; do
  IG_HOT_SAMPLE_STRIDE=$st timeout 900 python bench.py --config c3 --steps 6 --no-cpu-baseline --no-e2e > gpurun_out/s3s_bench_c3_$st.json 2> gpurun_out/s3s_bench_c3.err; echo rc=$?
done
python - <<'P'
import json
for st in [64,128,256,32]:
    try:
        j=json.load(open(f'gpurun_out/s3s_bench_c3_{st}.json'))
        print(st, round(j['value'],2), round(j['ms_per_step'],1), {k:round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k}, j['result_digest'])
    except Exception as e: print(st, 'ERR', e)
P
