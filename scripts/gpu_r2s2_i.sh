set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_count_all_paths.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -rf > gpurun_out/pytest_new.txt 2>&1; echo rc_new=$?
tail -2 gpurun_out/pytest_new.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_q5.json 2> gpurun_out/bench_q5.err; echo rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/hot6q5 python bench.py --profile-run > gpurun_out/ncu_q5.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/hot6q5.ncu-rep --page details > gpurun_out/hot6q5_details.txt 2>/dev/null
ncu -i gpurun_out/hot6q5.ncu-rep --page source --csv > gpurun_out/hot6q5_source.csv 2>/dev/null
rm -f gpurun_out/hot6q5.ncu-rep
gzip -f gpurun_out/*_source.csv
