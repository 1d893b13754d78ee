# call l: evidence on the current code: every config's bench line, the c3
# reference arm, the c3 launch list, full-size parity verbose
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python bench.py > gpurun_out/r19_bench_c3.json 2> gpurun_out/r19_bench_c3.err; echo rc_c3=$?
for c in c1 c2 c4 c5; do
  timeout 1200 python bench.py --config $c > gpurun_out/r19_bench_$c.json 2> gpurun_out/r19_bench_$c.err; echo rc_$c=$?
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r19_ref_c3.json 2> gpurun_out/r19_ref_c3.err; echo rc_ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r19_launches_c3.csv python bench.py --profile-run > gpurun_out/ncu_list.log 2>&1
echo rc_list=$?
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -v --durations=0 > gpurun_out/r19_fullsize.txt 2>&1; echo rc_full=$?
tail -15 gpurun_out/r19_fullsize.txt
