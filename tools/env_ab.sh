# A/B over environment settings: ENVS="A=1 B=2|A=3" (| separates variants)
IFS='|' read -ra VS <<< "${ENVS}"
for v in "" "${VS[@]}"; do
  env $v timeout 900 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/envab.log 2>&1
  echo "== [$v] rc=$?"
  tail -1 gpurun_out/envab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v})"
done
