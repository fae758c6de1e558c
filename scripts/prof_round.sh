# Round profile: plain bench, launch list (ncu, all kernels), full capture of the top kernels.
# usage: bash scripts/prof_round.sh <tag>
TAG=${1:-r1}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_cluster|k_assoc_points|k_accum_points|k_finalize|k_assemble_graph" -s 20 -c 5 -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo prof_rc=$?
