# Round profile capture (one gpurun call): GPU tests, the default bench line,
# timelines, the ncu launch list of one bench step and one full-set capture of
# K1 / K2 / the DDLMS block kernel.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 300 python tools/step_timeline.py --out gpurun_out/step_timeline.txt > /dev/null 2>&1
timeout 300 python tools/e2e_timeline.py --packed12 --out gpurun_out/e2e_timeline.txt > /dev/null 2>&1
timeout 600 python tools/ddlms_modes_bench.py > gpurun_out/modes.log 2>&1
export KK_DDLMS_GRAPH=0
python tools/prof_run.py 26 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kk_pairs_kernel|static_blocks_kernel|ddlms_block_kernel" -c 12 -o gpurun_out/prof_r2l python tools/prof_run.py 26 2 > gpurun_out/ncu_full.log 2>&1
python bench.py --steps 2 --warmup 1 --no-checks --no-64qam --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r2l.csv python bench.py --steps 2 --warmup 1 --no-checks --no-64qam --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
