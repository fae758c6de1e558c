for v in "" nocommit; do
  if [ -n "$v" ]; then export MIS_LIB_PATH=paper_1803_02009_b200/libmis_$v.so; else unset MIS_LIB_PATH; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/vb_$v.json 2> gpurun_out/vb_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/vb_$v.json')); print('v=$v', d['ms_per_step'], d['roofline_k3']['accum_points']['launch_ms'])"
done
