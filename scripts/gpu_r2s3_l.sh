# call l (session 3): ncu --set full of the c2 4-gram scatter with stall reasons and per-line counters
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py --config c2 --profile-run > gpurun_out/s3l_plain_c2.log 2>&1; echo rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_route_scatter -s 1 -c 1 -o gpurun_out/s3l_c2_scatter python bench.py --config c2 --profile-run > gpurun_out/s3l_ncu_c2.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/s3l_c2_scatter.ncu-rep --page details > gpurun_out/s3l_c2_scatter_details.txt 2>/dev/null
ncu -i gpurun_out/s3l_c2_scatter.ncu-rep --page raw --csv > gpurun_out/s3l_c2_scatter_raw.csv 2>/dev/null
ncu -i gpurun_out/s3l_c2_scatter.ncu-rep --page source --csv > gpurun_out/s3l_c2_scatter_source.csv 2>/dev/null
rm -f gpurun_out/s3l_c2_scatter.ncu-rep
gzip -f gpurun_out/s3l_c2_scatter_source.csv
timeout 900 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/s3l_bench_c2.json 2> gpurun_out/s3l_bench_c2.err; echo rc=$?
grep "timed step" gpurun_out/s3l_bench_c2.err
