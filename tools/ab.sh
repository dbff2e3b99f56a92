# A/B: default library vs variants under paper_2405_02187_b200/_build_<name>/ (bench --no-cpu, kernel split)
for v in "" ${VARIANTS:-}; do
  if [ -z "$v" ]; then lib=paper_2405_02187_b200/_build/libcsf_b200.so; name=default; else lib=paper_2405_02187_b200/_build_$v/libcsf_b200.so; name=$v; fi
  CSF_B200_LIB=$lib timeout 900 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/ab_$name.log 2>&1
  echo "== $name rc=$?"
  tail -1 gpurun_out/ab_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v})"
done
