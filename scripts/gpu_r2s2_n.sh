# call n: pooled one-shot sessions; parity subset; c1/c2/c3 lines
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_host_paths.py tests/test_gpu_long_grams.py tests/test_gpu_exact.py tests/test_gpu_once_direct.py tests/test_ref_unit_tests.py tests/test_gpu_cli.py -q -rf > gpurun_out/pytest_new.txt 2>&1; echo rc_new=$?
tail -3 gpurun_out/pytest_new.txt
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/r21_bench_$c.json 2> gpurun_out/r21_bench_$c.err; echo rc_$c=$?
done
