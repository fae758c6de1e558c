set -x
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assemble_points|k_solve" -s 6 -c 2 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
