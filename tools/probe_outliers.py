import sys, time, torch, numpy as np
sys.path.insert(0, ".")
import graphgen, paper_1911_10616_b200 as pkg
from cuda.bindings import runtime as rt
g = graphgen.config(2)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)
out = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
st = torch.cuda.current_stream(dev)
def reserved():
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    return int(v)
for i in range(3): pkg.evoke_orbits_edges(g.n, e, out=out, stream=st.cuda_stream)
torch.cuda.synchronize()
rows = []
for i in range(60):
    r0 = reserved()
    t0 = time.perf_counter()
    r = pkg.evoke_orbits_edges(g.n, e, out=out, stream=st.cuda_stream, return_stats=True, serial=(i % 2 == 1))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rows.append((r[1]["ms_total"], (t1 - t0) * 1e3, reserved() - r0, r0, i))
print("median", np.median([x[0] for x in rows]))
for x in sorted(rows, key=lambda x: -x[0])[:8]: print("lib %.1f host %.1f grow %d reserved %d call %d" % x)
print("growth calls", [(x[4], x[2]) for x in rows if x[2]])
