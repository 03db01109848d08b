// workmodel.cuh -- algorithmic work units of the enumeration passes,
// computed on request (evoke_options.flags & EVOKE_FLAG_WORKMODEL) by cheap reductions
// over the graph, never inside a timed step.  Units are the inner-loop visits each pass
// must make; bytes per unit are the data each visit must touch.
#pragma once
#include "common.cuh"

struct WorkUnits {
  u64 sum_d2;        // sum_v d(v)^2           : pair phases A and D (wedge visits)
  u64 sum_te2;       // sum_e T(e)^2           : pair phase B (x1), phase E (x2)
  u64 hub;           // hub-local inner visits : sum over (v,a) of sum_{b<a in tri(v,a)} T(v,b)
  u64 c5_wedge;      // cycles5 steps 1 and 6  : sum_w d(w) d+(w) + d-(w) d+(w)
  u64 c5_q;          // cycles5 steps 2 and 4  : sum_k d+(k)^2
  u64 tri_stream;    // triangle pass          : sum_{e=(a,b)} d+(b)
};

__global__ void k_units_vertex(DGraph g, WorkUnits* out) {
  u64 d2 = 0, c5w = 0, c5q = 0;
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
    const u64 d = dg_deg(g, v), dp = dg_dplus(g, v), dmi = d - dp;
    d2 += d * d;
    c5w += d * dp + dmi * dp;
    c5q += dp * dp;
  }
  d2 = warp_sum(d2); c5w = warp_sum(c5w); c5q = warp_sum(c5q);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out->sum_d2, d2);
    atomicAdd(&out->c5_wedge, c5w);
    atomicAdd(&out->c5_q, c5q);
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
