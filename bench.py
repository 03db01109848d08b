"""Benchmark: input edges/s for the full n x 73 5-vertex orbit matrix (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--impl reference]

A step is one full pass of the hot path (all SURVEY 8(a) rows: canonicalise, k-core order,
CSR, triangles, cliques, pair tables, hub-local, 5-cycles, gathers, combine) over the
synthetic graph of BASELINE configs[I-1] (default I=2, Chung-Lu n=1e5 -- configs[1], the
single-GPU workload).  `value` = cleaned undirected edges / step time with the input
already resident in HBM (device pointers through the C ABI); `e2e` = the same call with
pinned HOST buffers (H2D of the edge list and D2H of the n x 73 result inside the timed
region).  L2 is flushed (256 MiB write) between timed steps.  For N > 1 (torchrun), each
rank runs its shard of the same graph and the partials are summed with one NCCL reduce;
time = max over ranks (strong scaling: total work fixed).

--impl reference times the CPU oracle (test infrastructure; PAPER-defined plain ESU) on a
bounded sample of the same workload on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "input edges/s for full n×73 5-vertex orbit counts (wall, 1/2/4/8 B200); % HBM roof"
UNIT = "edges/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_sample(cfg_graph, target_deg=30):
    """Bounded sample of the workload for the CPU oracle: the subgraph of the config graph
    induced by its vertices of degree <= target_deg (same generator, tail cut)."""
    e = np.unique(np.sort(cfg_graph.edges.astype(np.int64), axis=1), axis=0)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=cfg_graph.n)
    keep = deg <= target_deg
    sub = e[keep[e[:, 0]] & keep[e[:, 1]]].astype(np.int32)
    return sub, f"config subgraph induced by vertices of degree <= {target_deg}: {sub.shape[0]} edges"


def run_cpu_oracle(cfg_graph, steps=1, target_deg=30):
    import oracle
    threads = os.cpu_count() or 1
    sub, desc = cpu_sample(cfg_graph, target_deg)
    oracle.orbits(8, [(0, 1)])  # build + load outside the timing
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.orbits(cfg_graph.n, sub, threads=threads)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    return {"value": sub.shape[0] / t, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": desc + f"; {t:.2f} s per run (plain ESU over all roots, OpenMP {threads} threads)"}


def bench_reference(args):
    """--impl reference: the CPU oracle as it stands, on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import graphgen
    g = graphgen.config(args.config)
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state beyond the library load done in run_cpu_oracle
    cb = run_cpu_oracle(g, steps=max(1, min(args.steps, 3)), target_deg=args.cpu_deg)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"config{args.config} CPU-oracle sample", "graph": g.name},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-deg", type=int, default=30)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)

    import torch
    import graphgen
    import paper_1911_10616_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    g = graphgen.config(args.config)
    edges_dev = torch.from_numpy(g.edges).to(dev)
    out_dev = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def step(stats=False):
        r = pkg.evoke_orbits_edges(g.n, edges_dev, out=out_dev, shard_index=rank, num_shards=world,
                                   stream=stream.cuda_stream, return_stats=stats)
        if world > 1:
            from paper_1911_10616_b200.parallel import reduce_partials
            reduce_partials(out_dev, dst=0)
        return r

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # ---- device-resident timed steps (CUDA events on the launching stream)
    times, pass_ms, launches, lib_launches = [], {}, 0, 0
    st_last = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if not os.environ.get("BENCH_NO_FLUSH"):  # diagnosis only: the contract flushes L2
                flush.fill_(1)
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1))
        # per-pass times and launch counts from the same call with statistics on (untimed:
        # the statistics add a host read after the result is complete)
        for _ in range(min(args.steps, 3)):
            flush.fill_(1)
            torch.cuda.synchronize()
            _, st = step(stats=True)
            torch.cuda.synchronize()
            for k, v in st["ms_pass"].items():
                pass_ms[k] = pass_ms.get(k, 0.0) + v / min(args.steps, 3)
            st_last = st
        launches = st_last["kernel_launches"] * args.steps
        lib_launches = st_last["library_launches"] * args.steps
    ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    m = st_last["m"]
    value = m / (ms / 1e3)

    # ---- e2e through the C ABI with pinned host buffers
    h_edges = torch.from_numpy(g.edges).pin_memory()
    h_out = torch.empty((g.n, 73), dtype=torch.int64).pin_memory()
    he = h_edges.numpy()
    ho = h_out.numpy().view(np.uint64)
    pkg.evoke_orbits_edges(g.n, he, out=ho, shard_index=rank, num_shards=world)
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        pkg.evoke_orbits_edges(g.n, he, out=ho, shard_index=rank, num_shards=world)
        if world > 1:
            t_ = torch.from_numpy(ho.view(np.int64)).to(dev)
            torch.distributed.reduce(t_, dst=0)
            h_out.copy_(t_.cpu())
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- roofline of the dominant pass (algorithmic bytes / its CUDA-event duration)
    peak, peak_src = load_peaks()
    _, wm = pkg.evoke_orbits_edges(g.n, edges_dev, out=out_dev, shard_index=rank, num_shards=world,
                                   stream=stream.cuda_stream, workmodel=True)
    torch.cuda.synchronize()
    roof = roofline(wm, pass_ms, peak, peak_src, step_ms=ms)
    # the same pass isolated: one untimed call with the concurrent passes run one after the
    # other (EVOKE_FLAG_SERIAL), so its duration is not stretched by sharing the GPU
    _, st_ser = pkg.evoke_orbits_edges(g.n, edges_dev, out=out_dev, shard_index=rank, num_shards=world,
                                       stream=stream.cuda_stream, return_stats=True, serial=True)
    torch.cuda.synchronize()
    iso_ms = st_ser["ms_pass"].get(roof["kernel"])
    if iso_ms and roof.get("algorithmic_bytes"):
        roof["isolated"] = {"ms": iso_ms, "achieved": roof["algorithmic_bytes"] / (iso_ms / 1e3) / 1e9,
                            "frac": roof["algorithmic_bytes"] / (iso_ms / 1e3) / 1e9 / peak,
                            "step_ms_serial": st_ser["ms_total"]}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms, "step_ms": [round(t, 3) for t in times],
                "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": f"BASELINE configs[{args.config - 1}]: {graphgen.CONFIG_NAMES[args.config]}",
                           "n": g.n, "m": m, "m_raw": int(g.edges.shape[0]), "triangles": st_last["triangles"],
                           "max_degree": st_last["max_degree"], "degeneracy": st_last["degeneracy"],
                           "wedges": st_last["wedges"], "parallelism": f"dp{world} (work-unit shards + NCCL reduce)",
                           "l2": "flushed between timed steps (256 MiB write)"},
                "e2e": {"value": m / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(g.edges.nbytes),
                        "d2h_bytes_per_step": int(g.n * 73 * 8),
                        "step_ms": [round(1e3 * t, 3) for t in e2e_times]},
                "gpu_launches": launches,
                "library_launches": lib_launches,
                "clocks": clk.summary(),
                "roofline": roof,
                "pass_ms": {k: round(v, 4) for k, v in pass_ms.items()}}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = run_cpu_oracle(g, steps=1, target_deg=args.cpu_deg)
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def traffic_of(pass_name):
    """DRAM bytes per launch of the pass's kernels from the committed ncu --set full capture
    (profiles/traffic.json, written by tools/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get("passes", {}).get(pass_name)
    except Exception:
        return None


def roofline(wm, pass_ms, peak_gbs, peak_src, step_ms=None):
    """Dominant pass and its achieved algorithmic GB/s: the
    library's work model (units x bytes/unit, one untimed call) over the pass's mean
    CUDA-event duration inside the timed steps."""
    compute_passes = {k: v for k, v in pass_ms.items() if k not in ("h2d", "d2h")}
    top = max(compute_passes, key=compute_passes.get)
    t = compute_passes[top] / 1e3
    bytes_ = wm["alg_bytes"].get(top, 0.0)
    # the pair, hub-local, 5-cycle and theta66/70 passes run concurrently: each pass time is
    # its own span, so the share is taken against the measured step, not the sum of passes
    base = {"bound": "hbm", "kernel": top, "peak": peak_gbs, "unit": "GB/s", "traffic": traffic_of(top),
            "ms": compute_passes[top], "peak_source": peak_src,
            "share_of_step": compute_passes[top] / step_ms if step_ms else None, "units": wm["units"]}
    if not bytes_ or t <= 0:
        base.update({"achieved": None, "frac": None})
        return base
    achieved = bytes_ / t / 1e9
    base.update({"achieved": achieved, "frac": achieved / peak_gbs, "algorithmic_bytes": bytes_})
    return base


if __name__ == "__main__":
    main()
