set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py 4 2 --serial > gpurun_out/timing4.log 2>&1; echo t4=$?
tail -25 gpurun_out/timing4.log
timeout 300 python tools/dev_units.py 3 > gpurun_out/units3.log 2>&1; cat gpurun_out/units3.log
timeout 300 python tools/dev_units.py 4 > gpurun_out/units4.log 2>&1; cat gpurun_out/units4.log
cat > /tmp/p3.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, graphgen, paper_1911_10616_b200 as pkg
g = graphgen.config(3); e = torch.from_numpy(g.edges).cuda()
for i in range(2): pkg.evoke_orbits_edges(g.n, e, serial=True); torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hub_process -s 1 -c 1 -o gpurun_out/prof3_hub -f python /tmp/p3.py > gpurun_out/prof3_hub.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/prof3_hub.ncu-rep > gpurun_out/prof3_hub.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof3_hub.ncu-rep 60 > gpurun_out/prof3_hub_lines.txt 2>&1
rm -f gpurun_out/prof3_hub.ncu-rep
head -50 gpurun_out/prof3_hub.txt
