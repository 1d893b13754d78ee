# call v (session 3): the driver's round-end sequence on the final code: GPU suite, smoke, both bench arms
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r26_pytest_gpu.txt
cat gpurun_out/r26_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r26_smoke.txt 2>&1; echo smoke rc=$?
timeout 1200 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/r26_ref_c3.json 2> gpurun_out/r26_ref_c3.err; echo ref rc=$?
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/r26_bench_c3.json 2> gpurun_out/r26_bench_c3.err; echo c3 rc=$?
grep "timed step" gpurun_out/r26_bench_c3.err
