# call n (session 3): full GPU suite + smoke + c3/c5/c1 lines on the final code
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r23_pytest_gpu.txt
cat gpurun_out/r23_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r23_smoke.txt 2>&1; echo smoke rc=$?
timeout 1500 python bench.py > gpurun_out/r23_bench_c3.json 2> gpurun_out/r23_bench_c3.err; echo c3 rc=$?
for c in c5 c1; do
  timeout 1500 python bench.py --config $c > gpurun_out/r23_bench_$c.json 2> gpurun_out/r23_bench_$c.err
  echo $c rc=$?
done
