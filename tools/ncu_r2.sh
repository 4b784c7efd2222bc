# Round-2 profile pass (run under gpurun from the repo root): a plain bench line, the launch list
# of the same command, and one ncu --set full capture of each dominant kernel (the first level-0
# slab of config 4 for the brick-resident engine, the coarsest multigrid solve, the LOD steps).
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_plain.json 2>gpurun_out/r2_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:resident3d_q4 -s 3 -c 1 -o gpurun_out/r2_q4 python tools/ncu_target.py hierarchy > gpurun_out/r2_ncu_q4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:mgcg -c 1 -o gpurun_out/r2_mg python tools/ncu_target.py hierarchy > gpurun_out/r2_ncu_mg.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"setup_brick" -s 3 -c 1 -o gpurun_out/r2_setup python tools/ncu_target.py hierarchy > gpurun_out/r2_ncu_setup.log 2>&1
echo done
