# Closing round-2 measurement set after the pair64 48-row table (run from the
# repo root under gpurun, ONE GPU) -> gpurun_out/r02f/: GPU tests, the bench
# lines the re-run kernel touches (4K fp32 headline, 4K fp64, 1080p N=32 at
# I=100/200, the 64-frame stream), the C5 sweep, a randomised stress, and ncu
# for pair64 (fp64 1080p, replayed re-runs at I=200) plus the 4K launch list.
O=gpurun_out/r02f
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2 > $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_4k_default.json 2> $O/e1.err
timeout 600 python bench.py --precision fp64 --no-cpu > $O/bench_4k_fp64.json 2> $O/e2.err
timeout 300 python bench.py --workload 1080p --support 32 --no-cpu > $O/bench_1080p_n32.json 2> $O/e3.err
timeout 300 python bench.py --workload 1080p --iterations 200 --no-cpu > $O/bench_1080p_n32_i200.json 2> $O/e4.err
timeout 300 python bench.py --workload stream64 --no-cpu > $O/bench_stream64.json 2> $O/e5.err
timeout 900 python tools/sweep.py > $O/sweep_c5_1080p.jsonl 2> $O/e6.err
timeout 900 python tools/stress_parity.py 400 3131 > $O/stress_parity_400_final.txt 2>&1
FSR_NO_CHUNK=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 40 --csv --log-file $O/launches_4k.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/launch_run.log 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:pair64_kernel -s 2 -c 1 -o /tmp/p64 python bench.py --workload 1080p --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_p64.log 2>&1
python tools/ncu_summary.py /tmp/p64.ncu-rep $O/pair64_1080p_fp64_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 900 $NCU -k regex:pair64_kernel -s 1 -c 1 -o /tmp/p64r python bench.py --workload 1080p --iterations 200 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_p64r.log 2>&1
python tools/ncu_summary.py /tmp/p64r.ncu-rep $O/pair64_rerun_replay_1080p_i200_ncu > /dev/null 2>&1
cat $O/pytest_gpu.txt
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], d.get('value'), e.get('value'), r.get('kernel'), r.get('main_ms'), r.get('frac'), d.get('dtype'))"; done
wc -l $O/*.jsonl
tail -n 1 $O/stress_parity_400_final.txt
for f in $O/*_ncu.txt; do echo "== $f"; head -14 $f | grep -E "time_duration|issue_active|warps_active|registers|stall share"; done
