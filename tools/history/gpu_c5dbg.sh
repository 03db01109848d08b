set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/wm.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, graphgen, paper_1911_10616_b200 as pkg
for c in [2, 4]:
    g = graphgen.config(c); e = torch.from_numpy(g.edges).cuda()
    _, st = pkg.evoke_orbits_edges(g.n, e, return_stats=True, serial=True)
    torch.cuda.synchronize()
PY
EVOKE_C5_HIST=1 timeout 300 python /tmp/wm.py 2>&1 | grep "c5 W"
for c in 2 4; do timeout 300 python tools/dev_timing.py $c 6 --serial 2>&1 | grep -E "wall|cycles5"; EVOKE_C5_HOT=0 timeout 300 python tools/dev_timing.py $c 6 --serial 2>&1 | grep -E "wall|cycles5"; done
