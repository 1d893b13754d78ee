# full ncu capture of kernels matching REGEX for one profile run: bash scripts/gpu_ncu_k.sh CONFIG SEQS REGEX TAG COUNT
CFG=$1; SEQS=$2; RX=$3; TAG=$4; CNT=${5:-3}
python bench.py --config $CFG --seqs $SEQS --profile-run > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$RX" -c $CNT -o gpurun_out/$TAG python bench.py --config $CFG --seqs $SEQS --profile-run > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$?
