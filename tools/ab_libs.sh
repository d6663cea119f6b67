# A/B the 4K main kernel across library builds (run under gpurun from the repo root):
#   bash tools/ab_libs.sh libfsr.so libfsr_a.so ...   (each twice, interleaved)
for r in 1 2; do
  for lib in "$@"; do
    FSR_LIBFSR=$PWD/paper_2202_13926_b200/$lib timeout 200 python bench.py --no-cpu --no-e2e --steps 10 ${BENCH_ARGS} 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],2), round(d['roofline']['main_ms'],3), d.get('rerun_blocks_per_step'))"
  done
done
