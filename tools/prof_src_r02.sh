O=gpurun_out/src
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warp16_kernel -s 2 -c 1 -o $O/w16 python bench.py --workload 1080p --support 16 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l1.log 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warpsegd_kernel -s 2 -c 1 -o $O/wsd4 python bench.py --workload 1080p --support 4 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l2.log 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:pair64_kernel -s 2 -c 1 -o $O/p64 python bench.py --workload 1080p --precision fp64 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l3.log 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warpn_kernel -s 2 -c 1 -o $O/wn24 python bench.py --workload 1080p --support 24 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l4.log 2>&1
FSR_NO_CHUNK=1 timeout 600 $NCU -k regex:warp32_kernel -s 2 -c 1 -o $O/w32 python bench.py --workload 1080p --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l5.log 2>&1
ls -la $O
