# A/B harness for kernel build variants (run from the repo root under gpurun):
#   make -C paper_2202_13926_b200/csrc EXTRA=-D... OUT=../libfsr_x.so, then
#   NOTEST=1 REPS=2 BENCH_ARGS="--support 16" bash tools/ab_bench.sh libfsr.so libfsr_x.so
# A/B kernel variants: pytest -m gpu on the default build (unless NOTEST=1), then
# the 4K bench per library, REPS rounds interleaved
[ "$NOTEST" = 1 ] || timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
for r in $(seq ${REPS:-1}); do
for lib in "$@"; do
  FSR_LIBFSR=$PWD/paper_2202_13926_b200/$lib timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ab_${lib}_$r.json 2> gpurun_out/ab_$lib.err
done
done
[ "$NOTEST" = 1 ] || cat gpurun_out/pytest_gpu.txt
for r in $(seq ${REPS:-1}); do
for lib in "$@"; do python -c "
import json,sys
d=json.load(open('gpurun_out/ab_${lib}_$r.json')); print('$lib', round(d['value'],3), round(d['roofline']['main_ms'],3), d['rerun_blocks_per_step'])" 2>&1 | tail -1; done; done
