# ncu captures of the round-2 kernels not in tools/profile_r02.sh: the segmented
# N=8 / N=4 kernels, warp16 and cta64 (1080p), pair64 with replay (1080p I=200).
O=gpurun_out/p02b
mkdir -p $O
NCU="ncu --set full --clock-control none"
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warpseg_kernel -s 2 -c 1 -o /tmp/ws8 python bench.py --workload 1080p --support 8 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l1.log 2>&1
python tools/ncu_summary.py /tmp/ws8.ncu-rep $O/warpseg8_1080p_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warpsegd_kernel -s 2 -c 1 -o /tmp/wsd4 python bench.py --workload 1080p --support 4 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l2.log 2>&1
python tools/ncu_summary.py /tmp/wsd4.ncu-rep $O/warpsegd4_1080p_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warp16_kernel -s 2 -c 1 -o /tmp/w16 python bench.py --workload 1080p --support 16 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l3.log 2>&1
python tools/ncu_summary.py /tmp/w16.ncu-rep $O/warp16_1080p_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 900 $NCU -k regex:cta64_kernel -s 2 -c 1 -o /tmp/c64 python bench.py --workload 1080p --support 64 --reducer linear --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l4.log 2>&1
python tools/ncu_summary.py /tmp/c64.ncu-rep $O/cta64_1080p_ncu > /dev/null 2>&1
FSR_NO_CHUNK=1 timeout 900 $NCU -k regex:pair64_kernel -s 1 -c 1 -o /tmp/p64r python bench.py --workload 1080p --iterations 200 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l5.log 2>&1
python tools/ncu_summary.py /tmp/p64r.ncu-rep $O/pair64_rerun_replay_1080p_i200_ncu > /dev/null 2>&1
for f in $O/*_ncu.txt; do echo "== $f"; head -14 $f | grep -E "time_duration|issue_active|warps_active|registers|stall share"; done
