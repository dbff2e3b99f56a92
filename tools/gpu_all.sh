# GPU box: tests + every bench workload (logs under gpurun_out/)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest=$rc; tail -2 gpurun_out/pytest_gpu.log | head -1
[ $rc -eq 0 ] || exit 1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --workload config3 --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
timeout 1500 python bench.py --workload config4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
timeout 900 python bench.py --workload config5 > gpurun_out/bench_c5.log 2>&1; echo bench5=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
for f in bench bench_c3 bench_c4 bench_c5 bench_ref; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value'],1), d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'))"; done
