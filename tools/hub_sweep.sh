set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for gi in 4194304 1048576 262144 65536; do
  EVOKE_HUB_GIANT=$gi EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py 3 2 --serial 2>&1 | grep -E "hub_local|giant"
done
EVOKE_HUB_SPLIT=256 timeout 300 python tools/dev_timing.py 3 2 --serial 2>&1 | grep -E "hub_local"
EVOKE_HUB_SPLIT=4096 timeout 300 python tools/dev_timing.py 3 2 --serial 2>&1 | grep -E "hub_local"
