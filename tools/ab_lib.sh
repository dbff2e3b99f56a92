# GPU box: A/B of two builds of the library (A = paper_2405_02187_b200/_build_a,
# built with `make BUILD=_build_a`; B = the default _build), alternating runs
# of the config-5 and config-2 benches; usage: bash tools/ab_lib.sh [rounds]
A=$PWD/paper_2405_02187_b200/_build_a/libcsf_b200.so
for i in $(seq 1 ${1:-3}); do
  for v in A B; do
    if [ $v = A ]; then export CSF_B200_LIB=$A; else unset CSF_B200_LIB; fi
    r5=$(timeout 600 python bench.py --workload config5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']), round(j['ms_per_step'],1))")
    r2=$(timeout 600 python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']), round(j['ms_per_step'],1))")
    echo "$v c5 $r5 c2 $r2"
  done
done
