// workmodel.cuh -- algorithmic work units of the enumeration passes,
// computed on request (evoke_options.flags & EVOKE_FLAG_WORKMODEL) by cheap reductions
// over the graph, never inside a timed step.  Units are the inner-loop visits each pass
// must make; bytes per unit are the data each visit must touch.
#pragma once
#include "common.cuh"

struct WorkUnits {
  u64 sum_d2;        // sum_v d(v)^2           : all wedges (context: what a plain pair pass walks)
  u64 sum_te2;       // sum_e T(e)^2           : pair diamonds (pass 1 x1, pass 2 x2)
  u64 hub;           // hub-local inner visits : sum over (v,a) of sum_{b<a in tri(v,a)} T(v,b)
  u64 c5_wedge;      // cycles5 steps 1 and 6  : w1 = sum_l sum_{w in N(l)} |Nsel(w)|
  u64 c5_q;          // cycles5 steps 2/4 and 3: w2 + w3 (see cycles5.cuh)
  u64 tri_stream;    // triangle pass          : sum_{e=(a,b)} d+(b)
  u64 pair_rwedge;   // pair wedges walked     : sum_u sum_{v in N(u), v != h*(u)} |N(v) & (u, n)|
  u64 pair_hwalk;    // h* term                : sum_u min(|N(h*) & (u, n)|, pair wedges of u)
};

// warp per vertex u (as a pair source and as a 5-cycle endpoint l = u)
__global__ void k_units_vertex(DGraph g, WorkUnits* out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  u64 d2 = 0, rw = 0, hw = 0, w1 = 0, w23 = 0;
  for (int64_t ui = gw; ui < g.n; ui += nw) {
    const int32_t u = (int32_t)ui;
    const int64_t r0 = g.rp[u], r1 = g.rp[u + 1], rm = r0 + g.dm[u];
    u64 s = 0, a1 = 0, a23 = 0;
    int32_t lmax = 0;
    for (int64_t t = r0 + lane; t < r1; t += 32) {
      const int32_t v = g.ci[t];
      const int32_t dv = dg_deg(g, v);
      // the part of N(v) above u (the pair pass forms each pair from its lower end)
      const int32_t e = g.eid[t];
      const int64_t pos = (g.esrc[e] == v) ? g.rp[v] + g.dm[v] + (e - g.orow[v]) : g.eslot_hi[e];
      const int32_t len = (int32_t)(g.rp[v + 1] - pos - 1);
      s += (u64)len;
      lmax = max(lmax, len);
      a1 += (u64)((v < u) ? dv : dv - g.dm[v]);
      if (t < rm) {
        const int64_t ok = g.orow[v], ok1 = g.orow[v + 1];
        a23 += (u64)(ok1 - ok);
        for (int64_t e2 = ok; e2 < ok1; e2++) {
          const int32_t j = g.ocol[e2];
          a23 += (u64)(g.orow[j + 1] - g.orow[j]);
        }
      }
    }
    s = warp_sum(s); a1 = warp_sum(a1); a23 = warp_sum(a23);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(FULL_MASK, lmax, o));
    if (lane == 0) {
      const u64 du = (u64)dg_deg(g, u);
      d2 += du * du;
      const u64 r = du > 0 ? s - (u64)lmax : 0;
      rw += r;
      hw += min((u64)lmax, r);  // h* term: a walk of N(h*) or a search per key, counted as the smaller
      w1 += a1;
      w23 += a23;
    }
  }
  if (lane == 0) {
    atomicAdd(&out->sum_d2, d2);
    atomicAdd(&out->pair_rwedge, rw);
    atomicAdd(&out->pair_hwalk, hw);
    atomicAdd(&out->c5_wedge, w1);
    atomicAdd(&out->c5_q, w23);
  }
}

__global__ void k_units_edge(DGraph g, const u32* __restrict__ Te, WorkUnits* out) {
  u64 t2 = 0, ts = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.m; e += (int64_t)gridDim.x * blockDim.x) {
    const u64 t = Te[e];
    t2 += t * t;
    ts += (u64)dg_dplus(g, g.edst[e]);
  }
  t2 = warp_sum(t2); ts = warp_sum(ts);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out->sum_te2, t2);
    atomicAdd(&out->tri_stream, ts);
  }
}

// thread per slot (v, a)
__global__ void k_units_hub(DGraph g, const u32* __restrict__ Te, WorkUnits* out) {
  u64 h = 0;
  const int64_t m2 = 2 * g.m;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t eva = g.eid[s];
    if (Te[eva] < 2) continue;
    const int32_t a = g.ci[s];
    const int32_t v = (g.esrc[eva] == a) ? g.edst[eva] : g.esrc[eva];
    const bool v_lo = g.esrc[eva] == v;
    for (int64_t r = g.foff[eva]; r < g.foff[eva + 1]; r++) {
      if (g.fx[r] >= a) continue;
      const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
      h += (u64)Te[evb];
    }
  }
  h = warp_sum(h);
  if ((threadIdx.x & 31) == 0) atomicAdd(&out->hub, h);
}
