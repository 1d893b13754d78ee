# Evidence for profiles/: the bench line, its kernel launch list, and one full
# ncu capture of the dominant kernel.  bash scripts/gpu_profiles.sh TAG
TAG=${1:-r01}
set -x
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launches.log 2>&1
python bench.py --profile-run > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_route_scatter|k_route_count|k_consume" -s 3 -c 3 -o gpurun_out/${TAG}_full python bench.py --profile-run > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
