B2="--config c5 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --seq-frames 0 --no-filter --no-lm"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_accum_points_umma" -s 10 -c 1 \
  -o gpurun_out/um5 python bench.py $B2 > gpurun_out/ncu_um4.log 2>&1; echo ncu=$?
