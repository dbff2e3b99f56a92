# GPU box: config-3 bench for each prebuilt library variant _variants/$v.so ($V).
for v in $V; do
  export CSF_B200_LIB=$PWD/_variants/$v.so
  timeout 900 python bench.py --workload config3 --no-cpu > gpurun_out/bench_c3_$v.log 2>&1
  tail -1 gpurun_out/bench_c3_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$v', 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],2), {x: round(k[x],2) for x in ('raycast','raycast_lift','icp','integrate')})"
done
