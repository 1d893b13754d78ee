# Round evidence on one B200: GPU suite, smoke, every config's bench line, the
# c2 launch list, and full ncu captures of the dominant kernels.
#   bash scripts/gpu_evidence.sh TAG
TAG=${1:-r12}
set -x
nvidia-smi -L
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/${TAG}_pytest_gpu.txt
cat gpurun_out/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo smoke rc=$?
for c in c2 c1 c3 c4 c5; do
  timeout 1500 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo $c rc=$?
done
# launch list of two c2 bench steps (per-launch device time, DRAM bytes, instructions)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo launches rc=$?
# full captures: c2 extension scatter (pass 4), c4 direct pass (pass 5), c5 count-all pass 5
ncu --set full --clock-control none --import-source on -k regex:k_route_scatter -s 1 -c 1 -o gpurun_out/${TAG}_c2_scatter python bench.py --config c2 --profile-run > gpurun_out/${TAG}_ncu1.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_once_direct -s 2 -c 1 -o gpurun_out/${TAG}_c4_direct python bench.py --config c4 --seqs 1024 --profile-run > gpurun_out/${TAG}_ncu2.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_count_all -s 2 -c 1 -o gpurun_out/${TAG}_c5_count_all python bench.py --config c5 --seqs 3584 --profile-run > gpurun_out/${TAG}_ncu3.log 2>&1; echo ncu3 rc=$?
echo done
