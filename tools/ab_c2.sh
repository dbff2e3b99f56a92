# GPU box: A/B of two library builds on the config-2 bench (A = _build_a,
# B = the default _build), alternating; usage: bash tools/ab_c2.sh [rounds] [workload]
A=$PWD/paper_2405_02187_b200/_build_a/libcsf_b200.so
WL=${2:-config2}
for i in $(seq 1 ${1:-3}); do
  for v in A B; do
    if [ $v = A ]; then export CSF_B200_LIB=$A; else unset CSF_B200_LIB; fi
    timeout 600 python bench.py --workload $WL --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$v', 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],2), {x: round(k[x],2) for x in ('raycast','raycast_lift','icp','integrate')})"
  done
done
