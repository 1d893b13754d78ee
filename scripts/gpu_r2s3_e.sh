# call e (session 3): ncu --set full of the c3 6-gram dense sweep and the c5 6-gram sparse sweep
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for ms in 50 1000 50 1000; do
  IG_CLOCK_POLL_MS=$ms timeout 900 python bench.py --config c3 --steps 8 --no-cpu-baseline --no-e2e > gpurun_out/s3e_bench_c3_poll$ms.json 2> gpurun_out/s3e_bench_c3_poll.err; echo rc=$?
  echo poll $ms; grep "timed step" gpurun_out/s3e_bench_c3_poll.err
done
timeout 600 python bench.py --profile-run > gpurun_out/s3e_plain_c3.log 2>&1; echo rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/s3e_c3_hot6 python bench.py --profile-run > gpurun_out/s3e_ncu_c3.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/s3e_c3_hot6.ncu-rep --page details > gpurun_out/s3e_c3_hot6_details.txt 2>/dev/null
ncu -i gpurun_out/s3e_c3_hot6.ncu-rep --page raw --csv > gpurun_out/s3e_c3_hot6_raw.csv 2>/dev/null
ncu -i gpurun_out/s3e_c3_hot6.ncu-rep --page source --csv > gpurun_out/s3e_c3_hot6_source.csv 2>/dev/null
rm -f gpurun_out/s3e_c3_hot6.ncu-rep
timeout 600 python bench.py --config c5 --seqs 16384 --profile-run > gpurun_out/s3e_plain_c5.log 2>&1; echo rc=$?
grep "profile run" gpurun_out/s3e_plain_c5.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/s3e_c5_hot6 python bench.py --config c5 --seqs 16384 --profile-run > gpurun_out/s3e_ncu_c5.log 2>&1
echo rc_ncu=$?
ncu -i gpurun_out/s3e_c5_hot6.ncu-rep --page details > gpurun_out/s3e_c5_hot6_details.txt 2>/dev/null
ncu -i gpurun_out/s3e_c5_hot6.ncu-rep --page raw --csv > gpurun_out/s3e_c5_hot6_raw.csv 2>/dev/null
rm -f gpurun_out/s3e_c5_hot6.ncu-rep
gzip -f gpurun_out/*_source.csv
head -3 gpurun_out/s3e_c5_hot6_details.txt
