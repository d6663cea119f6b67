# Round-2 measurement set (run from the repo root under gpurun) -> gpurun_out/r02/:
# GPU tests, whole-frame parity, the bench lines (4K fp32 headline, 4K fp64
# validation, 1080p at every support of the paper grid, stream of 64 frames),
# the reference arm, the C5 sweep and the paper-grid sweep, randomised stress.
O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2 > $O/pytest_gpu.txt
timeout 900 python -m pytest tests/test_gpu_fullframe.py -m gpu -q -s 2>&1 | grep -oE "N=[0-9]+ 1080p.*|fp(32|64) 1080p.*|[0-9]+ passed.*|[0-9]+ failed.*" > $O/fullframe_1080p.txt
timeout 600 python bench.py > $O/bench_4k_default.json 2> $O/e1.err
timeout 600 python bench.py --precision fp64 --no-cpu > $O/bench_4k_fp64.json 2> $O/e2.err
for s in 32 16 24 20 12 8 4; do
  timeout 300 python bench.py --workload 1080p --support $s --no-cpu > $O/bench_1080p_n$s.json 2> $O/e_$s.err
done
timeout 300 python bench.py --workload 1080p --support 64 --reducer linear --no-cpu > $O/bench_1080p_n64.json 2> $O/e_64.err
timeout 300 python bench.py --workload 1080p --iterations 200 --no-cpu > $O/bench_1080p_n32_i200.json 2> $O/e_i200.err
timeout 300 python bench.py --workload stream64 --no-cpu > $O/bench_stream64.json 2> $O/e4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_arm.json 2> $O/e5.err
timeout 900 python tools/sweep.py > $O/sweep_c5_1080p.jsonl 2> $O/e6.err
timeout 900 python tools/sweep.py --supports 4,8,24 --iterations 100,200,400 --argmax redux > $O/sweep_paper_grid_1080p.jsonl 2> $O/e7.err
timeout 900 python tools/stress_parity.py 400 2027 > $O/stress_parity_400_all_supports.txt 2>&1
timeout 600 python tools/stress_parity.py 200 2028 1 > $O/stress_parity_200_rho_gamma.txt 2>&1
cat $O/pytest_gpu.txt $O/fullframe_1080p.txt
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], d.get('value'), e.get('value'), r.get('kernel'), r.get('main_ms'), r.get('frac'), d.get('dtype'))"; done
wc -l $O/*.jsonl
for f in $O/stress_parity_*.txt; do tail -n 1 $f; done
