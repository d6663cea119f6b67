# Round-end measurement set (run from the repo root under gpurun): GPU tests, the
# bench lines copied to profiles/r01/, the reference arm and the C5 sweep.
# round-end measurement set -> gpurun_out/ (copied to profiles/r01 by hand)
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_4k_default.json 2> gpurun_out/e1.err
timeout 300 python bench.py --workload 1080p --no-cpu > gpurun_out/bench_1080p.json 2> gpurun_out/e2.err
timeout 300 python bench.py --workload 1080p --support 16 --no-cpu > gpurun_out/bench_1080p_n16.json 2> gpurun_out/e3.err
timeout 300 python bench.py --workload stream64 --no-cpu > gpurun_out/bench_stream64.json 2> gpurun_out/e4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_arm.json 2> gpurun_out/e5.err
timeout 900 python tools/sweep.py > gpurun_out/sweep_c5_1080p.jsonl 2> gpurun_out/e6.err
cat gpurun_out/pytest_gpu.txt
for f in bench_4k_default bench_1080p bench_1080p_n16 bench_stream64 bench_reference_arm; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('main_ms'), (d.get('cpu_baseline') or {}).get('value'))"; done
wc -l gpurun_out/sweep_c5_1080p.jsonl
