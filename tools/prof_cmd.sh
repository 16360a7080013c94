set -e
mkdir -p gpurun_out
export KK_DDLMS_GRAPH=0
python tools/prof_run.py 26 2 > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"kk_pairs_kernel|static_blocks_kernel|ddlms_block_kernel" -c 12 -o gpurun_out/prof_r2a python tools/prof_run.py 26 2 > gpurun_out/ncu_full.log 2>&1
python bench.py --steps 2 --warmup 1 --no-checks --no-64qam --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r2a.csv python bench.py --steps 2 --warmup 1 --no-checks --no-64qam --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
