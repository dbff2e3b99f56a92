# GPU box: (1) A/B of a candidate library build (_build) against HEAD
# (_build_a) on config 3 with its parity test — the candidate is kept only if
# it passes and is faster; (2) the round's measurement set; (3) the ncu
# summaries copied under gpurun_out/final/profiles and the .ncu-rep files
# removed (gpurun copies back at most 64 MiB).
mkdir -p gpurun_out/final/profiles
timeout 600 python -m pytest "tests/test_bench_configs.py::test_config3_all_pairs_vga" -m gpu -x -q > gpurun_out/cand_tests.log 2>&1
rc=$?
bash tools/ab_c2.sh 1 config3 > gpurun_out/cand_ab.log 2>&1
A=$(grep '^A ' gpurun_out/cand_ab.log | awk '{print $3}'); B=$(grep '^B ' gpurun_out/cand_ab.log | awk '{print $3}')
if [ "$rc" = 0 ] && python -c "import sys; sys.exit(0 if float('$B') > 1.005 * float('$A') else 1)"; then
  echo "candidate kept (A $A, B $B)"
else
  echo "candidate dropped (rc $rc, A $A, B $B)"; cp paper_2405_02187_b200/_build_a/libcsf_b200.so paper_2405_02187_b200/_build/libcsf_b200.so
fi
bash tools/gpu_round_end.sh > gpurun_out/round_end.log 2>&1
cp profiles/r02_ncu_*.csv profiles/traffic.json gpurun_out/final/profiles/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
cat gpurun_out/round_end.log
