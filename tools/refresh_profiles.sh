#!/bin/bash
# Round-end measurement pass on one B200 (run through gpurun from the repo
# root): the bench line, the ncu launch list of the same command (plain
# launches: ncu cannot see kernel nodes of graphs with conditional nodes),
# and ncu --set full captures of the top kernels.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
PM_USE_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-extras \
  > gpurun_out/launches.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_lj_step|k_verlet" \
  --launch-skip 20 --launch-count 12 -f -o gpurun_out/step_full python tools/prof_step.py --steps 200 \
  > gpurun_out/step_full.log 2>&1
echo "step capture rc=$?"
PM_USE_GRAPHS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sph_rates \
  --launch-skip 50 --launch-count 1 -f -o gpurun_out/sph_rates_full python tools/exp_sph_rate.py \
  > gpurun_out/sph_full.log 2>&1
echo "sph capture rc=$?"
PM_USE_GRAPHS=0 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:k_dem_step --launch-skip 320 --launch-count 1 -f -o gpurun_out/dem_step_full \
  python tools/dem_prof.py 300 50 > gpurun_out/dem_full.log 2>&1
echo "dem capture rc=$?"
