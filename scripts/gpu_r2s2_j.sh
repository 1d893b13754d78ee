# call j: split-way predicated hot lookups; guard tests; full GPU suite; c3 bench + ncu
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_q6.json 2> gpurun_out/bench_q6.err; echo rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/hot6q6 python bench.py --profile-run > gpurun_out/ncu_q6.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/hot6q6.ncu-rep --page details > gpurun_out/hot6q6_details.txt 2>/dev/null
ncu -i gpurun_out/hot6q6.ncu-rep --page source --csv > gpurun_out/hot6q6_source.csv 2>/dev/null
rm -f gpurun_out/hot6q6.ncu-rep
gzip -f gpurun_out/*_source.csv
timeout 900 python -m pytest tests/test_gpu_guard.py -q -rf > gpurun_out/pytest_guard.txt 2>&1; echo rc_guard=$?
tail -3 gpurun_out/pytest_guard.txt
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1; echo rc_pytest=$?
tail -8 gpurun_out/pytest_gpu.txt
