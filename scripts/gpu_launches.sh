# per-kernel launch list (device times) for one profile run: bash scripts/gpu_launches.sh CONFIG SEQS TAG
CFG=${1:-c2}; SEQS=${2:-256}; TAG=${3:-x}
python bench.py --config $CFG --seqs $SEQS --profile-run > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --config $CFG --seqs $SEQS --profile-run > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$?
