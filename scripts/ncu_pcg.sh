CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_pcg_cluster -s 5 -c 1 -o gpurun_out/pcg_$1 $CMD > gpurun_out/ncu_pcg.log 2>&1; echo ncu=$?
