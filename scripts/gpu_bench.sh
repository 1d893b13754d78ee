# usage: bash scripts/gpu_bench.sh  (on the GPU box, from the repo root)
set -x
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo rc=$?
tail -3 gpurun_out/bench_c1.err; cat gpurun_out/bench_c1.json
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?
tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
