# 4K pipeline shape sweep (run under gpurun): chunks x lanes, device and numpy-API calls
for cfg in "12 8" "8 8" "16 8" "12 6" "16 16" "12 12" "12 8"; do
  set -- $cfg
  echo "chunks $1 lanes $2: $(FSR_MAX_CHUNKS_RT=$1 FSR_LANES_RT=$2 python tools/device_probe.py 2>&1 | grep back-to-back) | $(FSR_MAX_CHUNKS_RT=$1 FSR_LANES_RT=$2 python tools/e2e_probe.py 2>&1 | grep 'api fresh')"
done
