set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/p3.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, graphgen, paper_1911_10616_b200 as pkg
g = graphgen.config(int(sys.argv[1])); e = torch.from_numpy(g.edges).cuda()
for i in range(int(sys.argv[2])): pkg.evoke_orbits_edges(g.n, e, serial=True); torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hub_heavy -s 1 -c 1 -o gpurun_out/prof3_hubh -f python /tmp/p3.py 3 2 > gpurun_out/prof3_hubh.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/prof3_hubh.ncu-rep > gpurun_out/prof3_hubh.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof3_hubh.ncu-rep 60 > gpurun_out/prof3_hubh_lines.txt 2>&1
rm -f gpurun_out/prof3_hubh.ncu-rep
head -60 gpurun_out/prof3_hubh.txt
EVOKE_C5_HIST=1 EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py 5 1 --warm 0 --serial > gpurun_out/timing5b.log 2>&1; echo t5=$?
grep -v "^\[evoke\] \(pair\|c5\) \(mid\|dense\|light\|heavy\) \(phases\|steps\)" gpurun_out/timing5b.log | tail -40
