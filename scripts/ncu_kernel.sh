# one full ncu capture of one launch of a kernel (regex) with dense warp sampling
#   bash scripts/ncu_kernel.sh <tag> <kernel-regex> [skip]
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:"$2" -s ${3:-5} -c ${4:-1} \
  -o gpurun_out/$1 $CMD > gpurun_out/ncu_$1.log 2>&1; echo ncu=$?
