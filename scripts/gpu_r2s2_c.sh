# call c: u32 extension tables (prefix-count bound), host streaming paths,
# library NCCL; full GPU suite, c3/c2 bench, ncu of a c3 extension sweep
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_paths.py tests/test_gpu_bench_collective.py tests/test_ref_unit_tests.py tests/test_gpu_exact.py -q -x -rf > gpurun_out/pytest_new.txt 2>&1; echo rc_new=$?
tail -5 gpurun_out/pytest_new.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc_c3=$?
tail -3 gpurun_out/bench_c3.err
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1; echo rc_pytest=$?
tail -8 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc_c2=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --profile-run > gpurun_out/ncu_list.log 2>&1
echo rc_list=$?
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_count_hot<1, 6' -c 1 -o gpurun_out/r2_c3_hot6 python bench.py --profile-run > gpurun_out/ncu_c3.log 2>&1
echo rc_ncu=$?
tail -3 gpurun_out/ncu_c3.log
for r in gpurun_out/r2_c3_hot6.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $r --page details > ${r%.ncu-rep}_details.txt 2>/dev/null
  ncu -i $r --page source --csv > ${r%.ncu-rep}_source.csv 2>/dev/null
done
gzip -f gpurun_out/*_source.csv gpurun_out/*_raw.csv
s=$(du -sm gpurun_out/r2_c3_hot6.ncu-rep | cut -f1); if [ "$s" -gt 30 ]; then rm -f gpurun_out/r2_c3_hot6.ncu-rep; fi
du -sh gpurun_out
