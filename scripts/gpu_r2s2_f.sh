# call f: branch-free queued sweep: parity subset + c3 bench + ncu source of the 6-gram sweep
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py -q -x -rf > gpurun_out/pytest_new.txt 2>&1; echo rc_new=$?
tail -2 gpurun_out/pytest_new.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; echo rc=$?
python -c "
import json; j=json.loads(open('gpurun_out/bench_q3.json').read().strip().splitlines()[-1]); print("q3", round(j['value'],2), round(j['ms_per_step'],1), j['result_digest'], {k: round(v,1) for k,v in j['step_breakdown_ms'].items() if 'pass' in k})"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/hot6q3 python bench.py --profile-run > gpurun_out/ncu_q2.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/hot6q3.ncu-rep --page details > gpurun_out/hot6q3_details.txt 2>/dev/null
ncu -i gpurun_out/hot6q3.ncu-rep --page source --csv > gpurun_out/hot6q3_source.csv 2>/dev/null
rm -f gpurun_out/hot6q3.ncu-rep
gzip -f gpurun_out/*_source.csv
