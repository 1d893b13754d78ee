# round 2, session 2, call a: GPU suite, c3 bench (driver default), c2 bench,
# reference arm, c3 launch list, one ncu --set full of the c3 counting kernels
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo rc_pytest=$?
tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc_c3=$?
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc_c2=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err; echo rc_ref=$?
python bench.py --profile-run > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --profile-run > gpurun_out/ncu_list.log 2>&1
echo rc_list=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_count_(hot|all)" -c 16 -o gpurun_out/r2_c3_count python bench.py --profile-run > gpurun_out/ncu_c3.log 2>&1
echo rc_ncu=$?
tail -3 gpurun_out/ncu_c3.log
