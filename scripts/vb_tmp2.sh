for v in "$@"; do
  if [ "$v" != "cur" ]; then export MIS_LIB_PATH=paper_1803_02009_b200/libmis_$v.so; else unset MIS_LIB_PATH; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 20 --no-lm > gpurun_out/vb_$v.json 2> gpurun_out/vb_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/vb_$v.json')); r=d['roofline_k3']; k=d['kernels_ms_per_step']; print('v=$v', d['ms_per_step'], 'e2e', d['e2e']['value'], 'K3a',r['assoc_points']['launch_ms'], 'K3b', r['accum_points']['launch_ms'], 'solve', d['roofline']['launch_ms'], 'fin', k.get('finalize'), 'pcg', d['pcg_phases_us_last_launch'].get('pcg'))"
done
