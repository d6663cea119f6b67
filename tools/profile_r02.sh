# ncu evidence for profiles/r02/ (run from the repo root under gpurun, ONE GPU):
# the launch list of the default bench command, and one --set full capture per
# kernel choice: warp32 with each argmax arm (shfl / smem / redux, 1080p, the
# paper's ablation), the fp64 kernels (pair64, warp16d, cta64d, warpnd) and the
# new supports' fp32 kernel (warpn, N=24).  Summaries via tools/ncu_summary.py.
O=gpurun_out/p02
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
FSR_NO_CHUNK=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 40 --csv --log-file $O/launches_4k.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/launch_run.log 2>&1
for am in redux shfl smem; do
  FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warp32_kernel -s 2 -c 1 -o /tmp/w32_$am python bench.py --workload 1080p --argmax $am --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_w32_$am.log 2>&1
  python tools/ncu_summary.py /tmp/w32_$am.ncu-rep $O/warp32_1080p_${am}_ncu > /dev/null 2>&1
done
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warp32_kernel -s 2 -c 1 -o $O/w32_4k python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_w32_4k.log 2>&1
python tools/ncu_summary.py $O/w32_4k.ncu-rep $O/warp32_ncu > /dev/null 2>&1
ncu -i $O/w32_4k.ncu-rep --page source --csv --print-source sass > $O/w32_4k_sass.csv 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:pair64_kernel -s 2 -c 1 -o /tmp/p64 python bench.py --workload 1080p --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_p64.log 2>&1
python tools/ncu_summary.py /tmp/p64.ncu-rep $O/pair64_1080p_fp64_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warp16d_kernel -s 2 -c 1 -o /tmp/w16d python bench.py --workload 1080p --support 16 --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_w16d.log 2>&1
python tools/ncu_summary.py /tmp/w16d.ncu-rep $O/warp16d_1080p_fp64_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 900 $NCU -k regex:cta64d_kernel -s 1 -c 1 -o /tmp/c64d python bench.py --workload 1080p --support 64 --reducer linear --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_c64d.log 2>&1
python tools/ncu_summary.py /tmp/c64d.ncu-rep $O/cta64d_1080p_fp64_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warpn_kernel -s 2 -c 1 -o /tmp/wn24 python bench.py --workload 1080p --support 24 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_wn24.log 2>&1
python tools/ncu_summary.py /tmp/wn24.ncu-rep $O/warpn24_1080p_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warpnd_kernel -s 2 -c 1 -o /tmp/wnd24 python bench.py --workload 1080p --support 24 --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_wnd24.log 2>&1
python tools/ncu_summary.py /tmp/wnd24.ncu-rep $O/warpnd24_1080p_fp64_ncu > /dev/null 2>&1


rm -f $O/w32_4k.ncu-rep
ls $O
for f in $O/*_ncu.txt; do echo "== $f"; head -12 $f | grep -E "time_duration|issue_active|warps_active|registers|stall share"; done
