# call m: inline rank-bitmap pass A/B, c1 with the raised hot threshold, c4 line
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IG_HOT_Q5=1 IG_HOT_MIN_TILES=1 timeout 900 python -m pytest tests/test_gpu_count_all_paths.py -q -x > gpurun_out/pytest_q5.txt 2>&1; echo rc_q5=$?
tail -1 gpurun_out/pytest_q5.txt
for env in "IG_X=0" "IG_HOT_Q5=1"; do
  env $env timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$env.json 2> gpurun_out/bench_$env.err; echo rc=$?
done
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r20_bench_c1.json 2> gpurun_out/r20_bench_c1.err; echo rc_c1=$?
timeout 1200 python bench.py --config c4 > gpurun_out/r20_bench_c4.json 2> gpurun_out/r20_bench_c4.err; echo rc_c4=$?
