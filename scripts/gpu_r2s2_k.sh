# call k: 256-bit bucket loads; queued rank-bitmap pass A/B; ncu of the 7-gram sweep
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py -q -x -rf > gpurun_out/pytest_new.txt 2>&1; echo rc_new=$?
tail -1 gpurun_out/pytest_new.txt
for env in "IG_X=0" "IG_HOT_Q5=1"; do
  env $env timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$env.json 2> gpurun_out/bench_$env.err; echo rc=$?
done
IG_HOT_Q5=1 timeout 600 python -m pytest tests/test_gpu_count_all_paths.py -q -x > gpurun_out/pytest_q5.txt 2>&1; echo rc_q5=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 9 -c 1 -o gpurun_out/hot7 python bench.py --profile-run > gpurun_out/ncu_7.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/hot7.ncu-rep --page details > gpurun_out/hot7_details.txt 2>/dev/null
ncu -i gpurun_out/hot7.ncu-rep --page source --csv > gpurun_out/hot7_source.csv 2>/dev/null
rm -f gpurun_out/hot7.ncu-rep
gzip -f gpurun_out/*_source.csv
