# Round profile of one bench config: plain bench, launch list (ncu, all kernels), full capture of the
# top kernels.  usage: bash scripts/prof_round.sh <tag> [config]
# then (here): python scripts/ncu_summary.py <tag> --round r2 --config <config>
TAG=${1:-r2}
CFG=${2:-c3}
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-lm --no-filter --seq-frames 0"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_cluster|k_solve|k_assoc_points|k_assoc_chunks|k_accum_points|k_finalize" -s 20 -c 8 -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo prof_rc=$?
