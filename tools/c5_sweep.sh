set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
for sc in 64 128 256 512; do for lb in 2 4 8; do
  echo "SHCAP=$sc LBPS=$lb"; EVOKE_C5_SHCAP=$sc EVOKE_C5_LBPS=$lb timeout 300 python tools/dev_timing.py 4 3 --serial 2>&1 | grep -E "cycles5"
done; done
