for r in 1 2; do for l in 8 12; do
  echo "lanes $l: $(FSR_LANES_RT=$l python tools/device_probe.py 2>&1 | grep back-to-back) | $(FSR_LANES_RT=$l python tools/e2e_probe.py 2>&1 | grep 'api fresh')"
done; done
FSR_LANES_RT=12 FSR_HOST_TRACE=1 FSR_CHUNK_TRACE=1 python tools/host_trace_probe.py 2>&1 | sed -n '/traced call/,$p'
