# ncu evidence for profiles/r01/ (run from the repo root under gpurun): launch list of
# the default bench command, --set full captures of warp32 and pair64, summaries.
# launch list of the default bench command + one full ncu capture of the 4K main kernel (unchunked)
FSR_NO_CHUNK=1 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 40 --csv --log-file gpurun_out/launches_4k.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/launch_run.log 2>&1
FSR_NO_CHUNK=1 ncu --set full --clock-control none --import-source on -k regex:warp32_kernel -s 2 -c 1 -o gpurun_out/w32_4k python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_run.log 2>&1
FSR_NO_CHUNK=1 ncu --set full --clock-control none --import-source on -k regex:pair64_kernel -s 2 -c 1 -o /tmp/p64_4k python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_run2.log 2>&1
python tools/ncu_summary.py gpurun_out/w32_4k.ncu-rep gpurun_out/warp32_ncu > gpurun_out/sum1.log 2>&1
python tools/ncu_summary.py /tmp/p64_4k.ncu-rep gpurun_out/pair64_ncu > gpurun_out/sum2.log 2>&1
ncu -i gpurun_out/w32_4k.ncu-rep --page source --csv --print-source sass > gpurun_out/w32_sass.csv 2>&1
ls -la gpurun_out | tail -12
# the other supports' main kernels at 1080p (bench's roofline for those lines)
FSR_NO_CHUNK=1 ncu --set full --clock-control none -k regex:warp16_kernel -s 2 -c 1 -o /tmp/w16 python bench.py --workload 1080p --support 16 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_run3.log 2>&1
FSR_NO_CHUNK=1 ncu --set full --clock-control none -k regex:cta64_kernel -s 2 -c 1 -o /tmp/c64 python bench.py --workload 1080p --support 64 --reducer linear --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_run4.log 2>&1
python tools/ncu_summary.py /tmp/w16.ncu-rep gpurun_out/warp16_ncu > gpurun_out/sum3.log 2>&1
python tools/ncu_summary.py /tmp/c64.ncu-rep gpurun_out/cta64_ncu > gpurun_out/sum4.log 2>&1
