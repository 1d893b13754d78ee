# Round-end evidence on one B200: the whole GPU suite, smoke, and the bench
# line of every BASELINE config.  bash scripts/gpu_round.sh TAG
TAG=${1:-r05}
set -x
nvidia-smi -L
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/${TAG}_pytest_gpu.txt
cat gpurun_out/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo smoke rc=$?
for c in c2 c1 c3 c4 c5; do
  timeout 1500 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo $c rc=$?
done
