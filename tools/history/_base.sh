set -x
for c in 2 4 3; do
  timeout 300 python tools/dev_timing.py $c 3 > gpurun_out/base_t$c.log 2>&1
  EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py $c 1 --serial > gpurun_out/base_s$c.log 2>&1
done
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/base_mem.txt
