# ncu captures of the counting kernels (one GPU). usage: bash scripts/gpu_ncu.sh TAG
TAG=${1:-prof}
python bench.py --config c1 --profile-run > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_count -c 2 -o gpurun_out/${TAG}_c1 python bench.py --config c1 --profile-run > gpurun_out/ncu_c1.log 2>&1
echo rc_c1=$?
python bench.py --config c2 --seqs 256 --profile-run > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_count -c 2 -o gpurun_out/${TAG}_c2 python bench.py --config c2 --seqs 256 --profile-run > gpurun_out/ncu_c2.log 2>&1
echo rc_c2=$?
tail -3 gpurun_out/plain_c1.log gpurun_out/plain_c2.log gpurun_out/ncu_c1.log gpurun_out/ncu_c2.log
