# Re-take the N=64 evidence after cta64d's 79-row W table (run from the repo root
# under gpurun, ONE GPU) -> gpurun_out/r02g/: GPU tests, the N=64 bench line,
# the N=64 fp64 line, the C5 sweep, the paper-grid sweep, ncu of cta64d.
O=gpurun_out/r02g
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2 > $O/pytest_gpu.txt
timeout 300 python bench.py --workload 1080p --support 64 --reducer linear --no-cpu > $O/bench_1080p_n64.json 2> $O/e1.err
timeout 300 python bench.py --workload 1080p --support 64 --reducer linear --precision fp64 --no-cpu > $O/bench_1080p_n64_fp64.json 2> $O/e2.err
timeout 900 python tools/sweep.py > $O/sweep_c5_1080p.jsonl 2> $O/e3.err
FSR_NO_CHUNK=1 timeout 900 $NCU -k regex:cta64d_kernel -s 1 -c 1 -o /tmp/c64d python bench.py --workload 1080p --support 64 --reducer linear --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_c64d.log 2>&1
python tools/ncu_summary.py /tmp/c64d.ncu-rep $O/cta64d_1080p_fp64_ncu > /dev/null 2>&1
cat $O/pytest_gpu.txt
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], d.get('value'), e.get('value'), r.get('kernel'), r.get('main_ms'), r.get('frac'), d.get('dtype'))"; done
head -14 $O/cta64d_1080p_fp64_ncu.txt | grep -E "time_duration|issue_active|warps_active|registers"
