# c3 probe: host info, c3 bench with kernel breakdown, one ncu --set full of count_all launches
set -x
nproc; free -g | head -2; lscpu | grep -i "model name"; df -h /tmp | tail -1
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-depth 1 > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err; echo rc=$?
tail -3 gpurun_out/c3_bench.err; cat gpurun_out/c3_bench.json
python bench.py --config c3 --profile-run > gpurun_out/plain_c3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_all -c 12 -o gpurun_out/r13_c3_count_all python bench.py --config c3 --profile-run > gpurun_out/ncu_c3.log 2>&1
echo rc_ncu=$?
tail -5 gpurun_out/ncu_c3.log
