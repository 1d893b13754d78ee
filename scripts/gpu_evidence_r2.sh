# Round-2 evidence on one B200: GPU suite, smoke, every config's bench line
# (c3 = the bench default), the reference arm on c3, the c3 launch list, and
# full ncu captures of the c3 6-gram sweep (dense variant) and the c5 6-gram
# sweep (sparse variant).   bash scripts/gpu_evidence_r2.sh TAG
TAG=${1:-r22}
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi -L
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/${TAG}_pytest_gpu.txt
cat gpurun_out/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo smoke rc=$?
timeout 1200 python bench.py --impl reference > gpurun_out/${TAG}_ref_c3.json 2> gpurun_out/${TAG}_ref_c3.err; echo ref rc=$?
timeout 1500 python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err; echo c3 rc=$?
for c in c1 c2 c4 c5; do
  timeout 1500 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo $c rc=$?
done
# launch list of one complete c3 run (per-launch device time, DRAM bytes, instructions)
python bench.py --profile-run > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c3.csv python bench.py --profile-run > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo launches rc=$?
gzip -f gpurun_out/${TAG}_launches_c3.csv
# full captures
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/${TAG}_c3_hot6 python bench.py --profile-run > gpurun_out/${TAG}_ncu1.log 2>&1; echo ncu1 rc=$?
ncu -i gpurun_out/${TAG}_c3_hot6.ncu-rep --page details > gpurun_out/${TAG}_ncu_c3_hot6.txt 2>/dev/null
ncu -i gpurun_out/${TAG}_c3_hot6.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_c3_hot6_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_c3_hot6.ncu-rep
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_count_hot --launch-skip 7 -c 1 -o gpurun_out/${TAG}_c5_hot6 python bench.py --config c5 --seqs 16384 --profile-run > gpurun_out/${TAG}_ncu2.log 2>&1; echo ncu2 rc=$?
ncu -i gpurun_out/${TAG}_c5_hot6.ncu-rep --page details > gpurun_out/${TAG}_ncu_c5_hot6_sparse.txt 2>/dev/null
ncu -i gpurun_out/${TAG}_c5_hot6.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_c5_hot6_sparse_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_c5_hot6.ncu-rep
echo done
