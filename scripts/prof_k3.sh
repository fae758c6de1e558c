# usage: bash scripts/prof_k3.sh <tag> <kernel-regex>
TAG=${1:-k3}; KRE=${2:-k_assemble_points}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 6 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo prof_rc=$?
