"""Benchmark: input edges/s for the full n x 73 5-vertex orbit matrix (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--impl reference]

A step is one full pass of the hot path (all SURVEY 8(a) rows: canonicalise, k-core order,
CSR, triangles, cliques, pair tables, hub-local, 5-cycles, gathers, combine) over the
synthetic graph of BASELINE configs[I-1].  Default I = 4: Holme-Kim n = 2e6, ~16M edges,
the largest configuration that fits one GPU (configs[4], R-MAT 23, is the 8-GPU one).
`value` = cleaned undirected edges / step time with the input already resident in HBM
(device pointers through the C ABI); `e2e` = the same work with the edge list in pinned
HOST memory and the n x 73 result read back to the host inside the timed region (N = 1: the
C-ABI call with host pointers; N > 1: H2D copy, the device call, the NCCL reduce, D2H on
rank 0).  L2 is flushed (256 MiB write) between timed steps.  For N > 1 every rank runs its
work-balanced shard of the same graph and the partials are summed with one NCCL reduce;
time = max over ranks (strong scaling: total work fixed).  Without WORLD_SIZE in the
environment, --gpus N > 1 starts the N ranks itself (torch.distributed.run, 127.0.0.1).
The config-2 workload (BASELINE configs[1], the round-1 headline) is timed too, as `config2`.

--impl reference times the CPU oracle (test infrastructure; PAPER-defined plain ESU) on a
bounded sample of the same workload on this box's host cores.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "input edges/s for full n×73 5-vertex orbit counts (wall, 1/2/4/8 B200); % HBM roof"
UNIT = "edges/s"
# oracle sample: the config's subgraph induced by its vertices of degree <= CPU_DEG[config]
# (same generator, tail cut), sized for ~10-30 s of oracle work on the box's host cores
CPU_DEG = {1: 10**9, 2: 30, 3: 12, 4: 14, 5: 12}


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


def cpu_sample(cfg_graph, target_deg):
    """Bounded sample of the workload for the CPU oracle: the subgraph of the config graph
    induced by its vertices of degree <= target_deg (same generator, tail cut)."""
    e = np.unique(np.sort(cfg_graph.edges.astype(np.int64), axis=1), axis=0)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=cfg_graph.n)
    keep = deg <= target_deg
    sub = e[keep[e[:, 0]] & keep[e[:, 1]]].astype(np.int32)
    return sub, f"config subgraph induced by vertices of degree <= {target_deg}: {sub.shape[0]} edges"


def run_cpu_oracle(cfg_graph, sub, desc, steps=1):
    import oracle
    threads = os.cpu_count() or 1
    oracle.orbits(8, [(0, 1)])  # build + load outside the timing
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.orbits(cfg_graph.n, sub, threads=threads)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    return {"value": sub.shape[0] / t, "unit": UNIT, "cores": threads, "kind": "oracle", "ms": t * 1e3,
            "sample": desc + f"; {t:.2f} s per run (plain ESU over all roots, OpenMP {threads} threads)"}


def bench_reference(args):
    """--impl reference: the CPU oracle as it stands, on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import graphgen
    g = graphgen.config(args.config)
    sub, desc = cpu_sample(g, args.cpu_deg or CPU_DEG[args.config])
    cb = run_cpu_oracle(g, sub, desc, steps=max(1, min(args.steps, 3)))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[{args.config - 1}]: {graphgen.CONFIG_NAMES[args.config]}",
                       "graph": g.name, "sample": desc, "timed_runs": max(1, min(args.steps, 3))},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: start the N ranks (one per GPU) here."""
    import torch
    if torch.cuda.device_count() < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but {torch.cuda.device_count()} "
                          f"visible GPUs (one rank per GPU)"}))
        return 1
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def l2_copy_peak(torch, dev):
    """L2-resident copy bandwidth (read + write bytes / s) of this device: two 24 MiB buffers
    (48 MiB of traffic per copy, well inside the 126 MB L2), best of 5 x 200 copies"""
    a = torch.empty(24 << 20, dtype=torch.uint8, device=dev)
    b = torch.empty_like(a)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * a.numel() * 200 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--extra-config", type=int, default=2, help="also time this config (0: none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-deg", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

    import torch
    import graphgen
    import paper_1911_10616_b200 as pkg
    from paper_1911_10616_b200.parallel import reduce_partials

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def timed_steps(g, edges_dev, out_dev, steps, warmup):
        def step(**kw):
            r = pkg.evoke_orbits_edges(g.n, edges_dev, out=out_dev, shard_index=rank, num_shards=world,
                                       stream=stream.cuda_stream, **kw)
            if world > 1:
                reduce_partials(out_dev, dst=0)
            return r
        for _ in range(max(warmup, 3)):
            step()
        torch.cuda.synchronize()
        times = []
        for _ in range(steps):
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
        return times, step

    g = graphgen.config(args.config)
    edges_dev = torch.from_numpy(g.edges).to(dev)
    out_dev = torch.empty((g.n, 73), dtype=torch.int64, device=dev)

    # ---- device-resident timed steps (CUDA events on the launching stream)
    pass_ms, st_last = {}, None
    with ClockSampler(local) as clk:
        times, step = timed_steps(g, edges_dev, out_dev, args.steps, args.warmup)
        # per-pass times and launch counts from the same call with statistics on (untimed:
        # the statistics add a host read after the result is complete)
        nstat = min(args.steps, 3)
        for _ in range(nstat):
            flush.fill_(1)
            torch.cuda.synchronize()
            _, st = step(return_stats=True)
            torch.cuda.synchronize()
            for k, v in st["ms_pass"].items():
                pass_ms[k] = pass_ms.get(k, 0.0) + v / nstat
            st_last = st
    launches = st_last["kernel_launches"] * args.steps
    lib_launches = st_last["library_launches"] * args.steps
    ms = max_over_ranks(float(np.mean(times)))
    m = st_last["m"]
    value = m / (ms / 1e3)

    # ---- work balance of the shards (estimates summed per shard by the library)
    balance = None
    if world > 1:
        own = torch.tensor([st_last["work_shard"][p] for p in pkg.SHARDED_PASSES], dtype=torch.float64, device=dev)
        allw = [torch.zeros_like(own) for _ in range(world)]
        torch.distributed.all_gather(allw, own)
        allw = torch.stack(allw).cpu().numpy()
        balance = {p: (float(allw[:, i].max() / allw[:, i].mean()) if allw[:, i].sum() > 0 else None)
                   for i, p in enumerate(pkg.SHARDED_PASSES)}

    # ---- e2e: inputs in pinned host memory, result read back to the host, every step
    h_edges = torch.from_numpy(g.edges).pin_memory()
    h_out = torch.empty((g.n, 73), dtype=torch.int64).pin_memory()
    he = h_edges.numpy()
    ho = h_out.numpy().view(np.uint64)

    def e2e_step():
        if world == 1:
            pkg.evoke_orbits_edges(g.n, he, out=ho)  # C ABI, host pointers: H2D + D2H inside
        else:
            ed = h_edges.to(dev, non_blocking=True)
            pkg.evoke_orbits_edges(g.n, ed, out=out_dev, shard_index=rank, num_shards=world,
                                   stream=stream.cuda_stream)
            reduce_partials(out_dev, dst=0)
            if rank == 0:
                h_out.copy_(out_dev)
            torch.cuda.synchronize()
    e2e_step()
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e2e_step()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(float(np.mean(e2e_times)))

    # ---- roofline of the dominant pass (algorithmic bytes / its CUDA-event duration)
    peak, peak_src = load_peaks()
    l2_peak = l2_copy_peak(torch, dev)
    _, wm = pkg.evoke_orbits_edges(g.n, edges_dev, out=out_dev, shard_index=rank, num_shards=world,
                                   stream=stream.cuda_stream, workmodel=True)
    torch.cuda.synchronize()
    # the passes isolated: one untimed call with the concurrent passes run one after the other
    # (EVOKE_FLAG_SERIAL), so a pass's duration is not stretched by sharing the GPU; the
    # dominant pass is the one with the longest isolated time
    _, st_ser = pkg.evoke_orbits_edges(g.n, edges_dev, out=out_dev, shard_index=rank, num_shards=world,
                                       stream=stream.cuda_stream, return_stats=True, serial=True)
    torch.cuda.synchronize()
    roof = roofline(wm, pass_ms, peak, peak_src, l2_peak, step_ms=ms, config=args.config,
                    dominant_by=st_ser["ms_pass"])
    iso_ms = st_ser["ms_pass"].get(roof["kernel"])
    if iso_ms and roof.get("algorithmic_bytes"):
        roof["isolated"] = {"ms": iso_ms, "achieved": roof["algorithmic_bytes"] / (iso_ms / 1e3) / 1e9,
                            "frac": roof["algorithmic_bytes"] / (iso_ms / 1e3) / 1e9 / peak,
                            "step_ms_serial": st_ser["ms_total"],
                            "pass_ms_serial": {k: round(v, 3) for k, v in st_ser["ms_pass"].items()}}
    del out_dev, edges_dev

    # ---- the round-1 workload (config 2), device-resident steps
    extra = None
    if args.extra_config and args.extra_config != args.config:
        g2 = graphgen.config(args.extra_config)
        e2d = torch.from_numpy(g2.edges).to(dev)
        o2d = torch.empty((g2.n, 73), dtype=torch.int64, device=dev)
        t2, step2 = timed_steps(g2, e2d, o2d, max(args.steps, 10), args.warmup)
        _, st2 = step2(return_stats=True)
        ms2 = max_over_ranks(float(np.mean(t2)))
        extra = {"workload": f"BASELINE configs[{args.extra_config - 1}]: {graphgen.CONFIG_NAMES[args.extra_config]}",
                 "m": st2["m"], "value": st2["m"] / (ms2 / 1e3), "unit": UNIT, "ms_per_step": ms2,
                 "step_ms": [round(t, 3) for t in t2]}
        del e2d, o2d

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms, "step_ms": [round(t, 3) for t in times],
                "step_spread": {"min": round(min(times), 3), "max": round(max(times), 3),
                                "cv": round(float(np.std(times) / np.mean(times)), 4)},
                "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": f"BASELINE configs[{args.config - 1}]: {graphgen.CONFIG_NAMES[args.config]}",
                           "n": g.n, "m": m, "m_raw": int(g.edges.shape[0]),
                           "edges_sha256": hashlib.sha256(g.edges.tobytes()).hexdigest(),
                           "triangles": st_last["triangles"], "max_degree": st_last["max_degree"],
                           "degeneracy": st_last["degeneracy"], "wedges": st_last["wedges"],
                           "parallelism": f"dp{world} (work-balanced unit shards + NCCL reduce)",
                           "l2": "flushed between timed steps (256 MiB write)"},
                "e2e": {"value": m / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(g.edges.nbytes),
                        "d2h_bytes_per_step": int(g.n * 73 * 8),
                        "step_ms": [round(1e3 * t, 3) for t in e2e_times]},
                "gpu_launches": launches,
                "library_launches": lib_launches,
                "clocks": clk.summary(),
                "roofline": roof,
                "pass_ms": {k: round(v, 4) for k, v in pass_ms.items()}}
        if balance is not None:
            line["work_balance_max_over_mean"] = balance
        if extra is not None:
            line["config2"] = extra
        if not args.no_cpu_baseline and world == 1:
            sub, desc = cpu_sample(g, args.cpu_deg or CPU_DEG[args.config])
            cb = run_cpu_oracle(g, sub, desc, steps=1)
            # the GPU on the oracle's exact sample, for a like-for-like ratio
            sd = torch.from_numpy(sub).to(dev)
            od = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
            for _ in range(3):
                pkg.evoke_orbits_edges(g.n, sd, out=od, stream=stream.cuda_stream)
            ts = []
            for _ in range(5):
                flush.fill_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                pkg.evoke_orbits_edges(g.n, sd, out=od, stream=stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            cb["gpu_same_sample"] = {"value": sub.shape[0] / (float(np.mean(ts)) / 1e3), "unit": UNIT,
                                     "ms": float(np.mean(ts)), "ratio_gpu_over_cpu": None}
            cb["gpu_same_sample"]["ratio_gpu_over_cpu"] = cb["gpu_same_sample"]["value"] / cb["value"]
            line["cpu_baseline"] = cb
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def traffic_of(pass_name, config):
    """DRAM bytes per launch of the pass's kernels from the committed ncu --set full capture
    (profiles/traffic.json, written by tools/ncu_traffic.py) when it was taken on this config,
    or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        if d.get("config") != config:  # a capture of another config (or of unknown config) says nothing here
            return None
        return d.get("passes", {}).get(pass_name)
    except Exception:
        return None


def roofline(wm, pass_ms, peak_gbs, peak_src, l2_gbs, step_ms=None, config=None, dominant_by=None):
    """Dominant pass and its achieved algorithmic GB/s: the
    library's work model (units x bytes/unit, one untimed call) over the pass's mean
    CUDA-event duration inside the timed steps; against the measured HBM copy bandwidth and,
    as a second denominator, the L2-resident copy bandwidth measured here."""
    compute_passes = {k: v for k, v in pass_ms.items() if k not in ("h2d", "d2h")}
    rank_by = {k: v for k, v in (dominant_by or compute_passes).items() if k in compute_passes}
    top = max(rank_by, key=rank_by.get)
    t = compute_passes[top] / 1e3
    bytes_ = wm["alg_bytes"].get(top, 0.0)
    # the pair, hub-local, 5-cycle and theta66/70 passes run concurrently: each pass time is
    # its own span, so the share is taken against the measured step, not the sum of passes
    base = {"bound": "hbm", "kernel": top, "peak": peak_gbs, "unit": "GB/s", "traffic": traffic_of(top, config),
            "ms": compute_passes[top], "peak_source": peak_src,
            "share_of_step": compute_passes[top] / step_ms if step_ms else None, "units": wm["units"]}
    if not bytes_ or t <= 0:
        base.update({"achieved": None, "frac": None})
        return base
    achieved = bytes_ / t / 1e9
    if base["traffic"]:
        # DRAM bytes the pass's kernels actually moved (ncu capture on this config) over the
        # pass time: how close the random sector traffic runs to the HBM peak
        base["traffic_gbs"] = base["traffic"] / t / 1e9
        base["traffic_frac"] = base["traffic_gbs"] / peak_gbs
        base["traffic_over_algorithmic"] = base["traffic"] / bytes_
    base.update({"achieved": achieved, "frac": achieved / peak_gbs, "algorithmic_bytes": bytes_,
                 "l2": {"peak": l2_gbs, "unit": "GB/s", "frac": achieved / l2_gbs,
                        "peak_source": "measured here: L2-resident copy (2 x 24 MiB buffers, read + write bytes)"}})
    return base


if __name__ == "__main__":
    main()
