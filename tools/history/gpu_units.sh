# developer: longest single unit of every heavy persistent kernel (EVOKE_DEBUG) on configs 3, 4, 5
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in 4 3 5; do
  EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py $c 1 --warm 0 --serial > gpurun_out/units$c.log 2>&1; echo t$c=$?
  grep "units\|c5 big\|endpoints\|tiers\|items\|wall" gpurun_out/units$c.log
done
