#!/usr/bin/env python
"""Headline benchmark of the B200 all-pairs IDW hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

Workload (default, BASELINE.json north_star): C3 = 1,048,576 data x 1,048,576
query points, p = 2, fp32, AoaS layout, tiled kernel (K2), FAST mode, inputs
from the reference's splitmix64 generator (data seed 0, query seed 1).  One
step = one whole job: broadcast of the data buffers from rank 0 (N > 1), every
rank's query shard through K2 + fix-up, gather of the predictions.

`value` is whole-job pairs/s with inputs resident in HBM, each step one replay
of a CUDA-graph plan of the call (idw_plan_*; CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks); `e2e`
is the same metric through the public drop-in API (`run_tiled` on host arrays:
H2D of store + queries and D2H of the predictions inside the timed region).
`roofline` relates k_tiled's own device time to the MUFU reciprocal roofline
measured by a probe kernel on the same GPU; `cpu_baseline` times the oracle's
C port of the reference loop on this host's cores over a bounded query sample.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port; the reference package itself cannot travel to the GPU box) on
all host threads, on the same config and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GPairs/s (data×query distance-weights/sec) fp32/fp64 at 1/2/4/8 B200; % of MUFU roofline"
K = 1024
CONFIGS = {
    # name: (n, m, layout, precision, variant, p, description)
    "c1": (10 * K, 10 * K, "soa", "single", "tiled", 2.0, "C1: 10K x 10K, p=2, fp32, SoA"),
    "c2": (100 * K, 100 * K, "aoas", "single", "tiled", 2.0, "C2: 100K x 100K, p=2, fp32, AoaS"),
    "c3": (1024 * K, 1024 * K, "aoas", "single", "tiled", 2.0,
           "C3: 1M data x 1M queries, p=2, fp32, AoaS, tiled (K2)"),
    "c4": (1024 * K, 1024 * K, "soa", "double", "nested_improved", 3.5,
           "C4: 1M x 1M, p=3.5, fp64, SoA, split-reduce (K3)"),
    "c5": (10240 * K, 100 * K, "aoas", "single", "tiled", 2.0,
           "C5: 10M data x 100K queries, p=2, fp32, AoaS, tiled (K2, chunked data)"),
}
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
SHARD_ALIGN = 256


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--mode", choices=("fast", "exact"), default="fast")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    # test hooks for the multi-rank path on a single-GPU box (not used by the driver)
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl")
    ap.add_argument("--device-override", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.lines: list[str] = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", gpu_id, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
def make_inputs(cfg_name):
    import numpy as np

    import paper_1402_4986_b200 as il

    n, m, layout, prec, variant, p, desc = CONFIGS[cfg_name]
    x, y, z = il.generate_cloud_arrays(n, 0)
    qx, qy, _ = il.generate_cloud_arrays(m, il.query_seed(0))
    store = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(layout), il.Precision(prec))
    return store, np.column_stack([qx, qy])


def cpu_sample(store, queries, p, seconds: float, threads: int):
    """Time the oracle port (run_naive semantics, all host threads) on a
    bounded query sample sized for ~`seconds` of CPU work."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    n = store.count
    m0 = max(threads * 16, 64)
    t0 = time.perf_counter()
    oracle.predict_mt(store, queries[:m0], p, threads=threads)
    dt0 = max(time.perf_counter() - t0, 1e-6)
    msub = int(min(queries.shape[0], max(m0, m0 * seconds / dt0)))
    msub = max(threads, (msub // threads) * threads)
    t1 = time.perf_counter()
    oracle.predict_mt(store, queries[:msub], p, threads=threads)
    dt = time.perf_counter() - t1
    return n * msub / dt / 1e9, msub, dt


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU (oracle port)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    import refinputs  # oracle/: inputs built without the product package

    n, m, layout, prec, variant, p, desc = CONFIGS[args.config]
    store, queries = refinputs.bench_inputs(n, m, layout, prec)
    threads = oracle.max_threads()
    # size one step for ~6 s of CPU work
    m0 = threads * 16
    t0 = time.perf_counter()
    oracle.predict_mt(store, queries[:m0], p, threads=threads)
    per_q = max(time.perf_counter() - t0, 1e-6) / m0
    msub = max(threads, int(6.0 / per_q) // threads * threads)
    msub = min(msub, m)
    for _ in range(args.warmup):
        oracle.predict_mt(store, queries[:msub], p, threads=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle.predict_mt(store, queries[:msub], p, threads=threads)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    value = n * msub * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GPairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if prec == "single" else "f64", "data": "synthetic splitmix64 (generate_cloud_arrays seeds 0/1)",
        "config": {"workload": desc, "n": n, "m": m, "layout": layout, "precision": prec, "variant": "naive (CPU)",
                   "p": p, "sample_queries_per_step": msub},
        "cpu_baseline": {"value": value, "unit": "GPairs/s", "cores": threads, "kind": "port",
                         "sample": f"{n} data x {msub} queries per step (oracle/idw_oracle.c predict_block, "
                                   f"{threads} pthreads, 256-query blocks)"},
        "e2e": {"value": value, "unit": "GPairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    # the arm must not have touched the product (its package or its library)
    imported = sorted(k for k in sys.modules if k.startswith("paper_1402_4986_b200"))
    try:
        mapped = "libidw_b200" in Path("/proc/self/maps").read_text()
    except OSError:
        mapped = False
    if imported or mapped:
        raise SystemExit(f"reference arm touched the product: modules={imported} libidw_b200 mapped={mapped}")
    line["product_loaded"] = False
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch

    import paper_1402_4986_b200 as il
    from paper_1402_4986_b200 import _capi
    from paper_1402_4986_b200.device import DevicePlan, DeviceStore
    from paper_1402_4986_b200.partition import QueryShardedRunner, StoreMeta, shard_bounds

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    if args.device_override is not None:
        local = args.device_override
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    n, m, layout, prec, variant, p, desc = CONFIGS[args.config]
    params = il.Params(p)
    cfg = il.ExecConfig(mode=args.mode, device=local)
    tdt = torch.float32 if prec == "single" else torch.float64

    # ---- inputs: data built on rank 0 and replicated by broadcast; each rank
    # holds its query shard in HBM before the timed region starts.
    store, queries = make_inputs(args.config) if rank == 0 or world == 1 else (None, None)
    if queries is None:
        qx64, qy64, _ = il.generate_cloud_arrays(m, il.query_seed(0))
        queries = np.column_stack([qx64, qy64])
    lo, hi = shard_bounds(m, world, rank, SHARD_ALIGN)
    npdt = np.float32 if prec == "single" else np.float64
    qx_l = torch.from_numpy(np.ascontiguousarray(queries[lo:hi, 0].astype(npdt))).to(dev)
    qy_l = torch.from_numpy(np.ascontiguousarray(queries[lo:hi, 1].astype(npdt))).to(dev)
    out_l = torch.empty(hi - lo, dtype=tdt, device=dev)

    if world > 1:
        runner = QueryShardedRunner(dist, dev, align=SHARD_ALIGN)
        meta = StoreMeta(layout, prec, n, [b.nbytes for b in store.buffers]) if rank == 0 else None
        meta = runner.broadcast_meta(meta)
        src_bufs = DeviceStore(store, local).tensors if rank == 0 else None
        bufs = runner.broadcast_buffers(src_bufs, meta)
        dstore = DeviceStore.from_tensors(il.LayoutKind(layout), il.Precision(prec), n, bufs, meta.nbytes, local)
    else:
        runner = None
        dstore = DeviceStore(store, local)
        bufs = dstore.tensors
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches = [0]

    # One CUDA-graph plan per timed step (idw_plan: bbox pre-pass + variant
    # kernels + fix-up captured once, replayed with one graph launch); each
    # plan's timing event nodes then hold its own step's kernel time.
    plans = [DevicePlan(dstore, qx_l, qy_l, out_l, params, cfg, variant) for _ in range(max(args.steps, 1))]

    def step(plan):
        if runner is not None:
            for t in bufs:  # the data replication collective (NVLink/NVSwitch)
                dist.broadcast(t, src=0)
        plan.launch(stream)
        launches[0] += plan.launches
        if runner is not None:
            runner.gather(out_l, m)

    # ---- MUFU roofline probe (same GPU, just before the timed region)
    probe_rate, probe_hz = _capi.mufu_peak(local)
    for w in range(max(args.warmup, len(plans))):  # every plan replays at least once before timing
        step(plans[w % len(plans)])
        flush.zero_()
    torch.cuda.synchronize(dev)
    props = torch.cuda.get_device_properties(dev)
    gpu_id = str(getattr(props, "uuid", local))
    if gpu_id and not gpu_id.startswith("GPU-") and len(gpu_id) == 36:
        gpu_id = "GPU-" + gpu_id
    sampler = ClockSampler(gpu_id)
    time.sleep(0.3)
    launches[0] = 0
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # One event pair per step on the launching stream; the L2 flush (256 MiB
    # write, > 126 MB L2) runs between steps, outside the timed intervals, and
    # nothing synchronises the host inside the loop.
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        ev[k][0].record(stream)
        step(plans[k])
        ev[k][1].record(stream)
        flush.zero_()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    ms_local = sum(a.elapsed_time(b) for a, b in ev)
    kern = [pl.kernel_ms() for pl in plans[:args.steps]]  # event nodes inside each step's graph
    ms = ms_local
    if dist is not None:
        t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_pairs = float(n) * float(m)
    value = total_pairs * args.steps / (ms * 1e-3) / 1e9
    ms_step = ms / args.steps

    # ---- roofline of the dominant kernel (k_tiled / k_nested), this rank
    kmain = statistics.mean(k[0] for k in kern)
    kfix = statistics.mean(k[1] for k in kern)
    pairs_launch = float(n) * float(hi - lo)
    achieved = pairs_launch / (kmain * 1e-3) / 1e9
    sms = props.multi_processor_count
    mufu_per_pair = 1 if p == 2.0 else 2
    run_clock_peak = None
    if clocks.get("sm_mhz"):
        run_clock_peak = sms * 16 * clocks["sm_mhz"] * 1e6 / mufu_per_pair / 1e9
    peak = probe_rate / mufu_per_pair / 1e9
    if prec == "double":
        # FP64-pipe bound: DP ops per pair of the FAST fp64 loop (SASS):
        # p = 2: 2 DADD + DMUL + DFMA (d2) + 3 DFMA (rcp correction) + DADD + DFMA = 9;
        # p = 3.5 / 3: 6 base + t^2, t^4, residual e = 1 - d2 t^4, t^jq (2 / 1 DMUL),
        # series (1 + a e + b e^2) folded into w = fma(t^jq, (a + b e) e, t^jq) (3)
        # = 14 / 13 (the d2^(-1/4) seed is fp32 MUFU work, not DP)
        dp_ops = {2.0: 9, 3.5: 14, 3.0: 13}.get(p, 50)
        mhz = clocks.get("sm_mhz") or 1965.0
        peak = sms * 64 * mhz * 1e6 / dp_ops / 1e9  # nominal 64 DP lanes/clk/SM (62 measured)
        run_clock_peak = peak
    if variant == "tiled":
        kname = "k_tiled_chunks" if args.mode == "fast" else "k_tiled"
    else:  # split-reduce: the warp-team kernel for FAST at 32 <= G <= 1024
        kname = "k_nested_warps" if args.mode == "fast" else "k_nested"
    roof = {
        "bound": "mufu" if prec == "single" else "fp64",
        "achieved": achieved,
        "peak": peak,
        "unit": "GPairs/s",
        "frac": achieved / peak,
        "traffic": None,
        "kernel": kname,
        "kernel_ms": kmain,
        "fixup_ms": kfix,
        "peak_source": "measured: idw_mufu_peak probe (independent rcp.approx chains on all "
                       f"{sms} SMs) just before the timed region; nominal 16 MUFU lanes/clk/SM",
        "peak_at_run_clock": run_clock_peak,
        "frac_at_run_clock": achieved / run_clock_peak if run_clock_peak else None,
        "algorithmic_unit": "one (query, data) pair = 1 rcp + 2 sums; n*m_shard pairs per launch",
    }
    if prec == "double":
        roof["peak_source"] = (f"FP64 pipe: {sms} SMs x 64 DP lanes/clk x run clock / {dp_ops} DP ops per pair "
                               "(DFMA measured 62/clk/SM in tools/microbench.cu)")
        # BASELINE.md §3 states the fp64 rooflines with the textbook arithmetic:
        # 10 DP instr/pair for p = 2, 6 + D_pow for general p, D_pow = 47 DP
        # instructions on the fast path of CUDA 12.9 exp2(wexp * log2(d2)) in
        # double (SASS of a probe kernel: 28 for log2, 19 for the multiply and
        # exp2).  The kernel's reformulated arithmetic needs fewer.
        base_ops = 10 if p == 2.0 else 6 + 47
        base_peak = sms * 64 * mhz * 1e6 / base_ops / 1e9
        roof["baseline_definition"] = {"dp_ops_per_pair": base_ops, "peak": base_peak, "frac": achieved / base_peak,
                                       "note": "BASELINE.md section 3 roofline; peak/frac above use the kernel's "
                                               f"own {dp_ops} DP ops per pair"}
    elif p == 2.0 and args.mode == "fast" and variant == "tiled":
        # The BASELINE roofline charges one MUFU reciprocal per pair.  k_tiled_chunks
        # computes one of its four packed query pairs with a shared reciprocal
        # (r = 1/(a*b), 1/a = b*r, 1/b = a*r), i.e. 7 MUFU per 8 pairs, so it
        # can pass that line; its own MUFU ceiling is peak * 8/7 (and the
        # FMA pipe, which carries the shared-reciprocal products, binds close
        # to it: 51 fp32 lane-ops per 8 pairs -> 20.1 pairs/clk/SM).
        mix_peak = peak * 8.0 / 7.0
        roof["kernel_mix_bound"] = {
            "mufu_per_pair": 7.0 / 8.0, "peak": mix_peak, "frac": achieved / mix_peak,
            "note": "MUFU ceiling of k_tiled_chunks' own instruction mix (shared reciprocal for 1 of 4 query pairs)"}
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # Algorithmic (compulsory) bytes of one launch: the store, the cast query
    # coordinates in, the predictions out -- n*S_rec + 3*m_shard*e.
    e_sz = 4 if prec == "single" else 8
    srec = {"soa": 3 * e_sz, "aos": 3 * e_sz, "aoas": 4 * e_sz, "soaos": 32, "hybrid": 24}[layout]
    roof["algorithmic_bytes"] = float(n * srec + 3 * (hi - lo) * e_sz)
    # DRAM traffic of the dominant kernel from the committed ncu --set full
    # capture of the same configuration (profiles/r2, tools/gpu_r2_profiles.sh)
    caps = {"c1": "prof_c1", "c2": "prof_c2", "c3": "prof_c3", "c5": "prof_c5"}  # C4's capture is 1M x 16K
    prof = ROOT / "profiles" / "r2" / f"{caps.get(args.config, '-')}.raw.csv"
    if prof.exists() and args.mode == "fast" and world == 1:
        import csv

        rows = list(csv.reader(open(prof)))
        kcol = rows[0].index("Kernel Name")
        row = next((r for r in rows[2:] if r[kcol].split("<")[0].split()[-1] == kname), None)
        d = dict(zip(rows[0], row)) if row else {}
        u = dict(zip(rows[0], rows[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        try:
            rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
            wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
            roof["traffic"] = rd + wr
            roof["traffic_read"] = rd
            roof["traffic_write"] = wr
            roof["traffic_source"] = f"{prof.relative_to(ROOT)} (ncu --set full, one {kname} launch, same config)"
            if kname == "k_tiled_chunks":
                roof["traffic_note"] = (
                    "chunk partials live in an L2-resident ring of group slots (recycled after each group's fold); "
                    "a store larger than L2/4 (C5) is swept by bands of query groups, so HBM streams it once per "
                    "band and the band's partials are written back")
        except (KeyError, ValueError):
            pass

    # ---- e2e through the public drop-in API (host buffers, blocking).  At
    # N > 1 the drop-in's own multi-GPU form runs: rank 0 makes ONE run_*
    # call over ExecConfig(devices=(0..N-1)) -- the store host->device once,
    # the peer-copy broadcast tree, N query shards on N GPUs, each shard
    # copied into its slice of the result -- while the other ranks wait at a
    # barrier (their GPUs are the call's devices 1..N-1).
    e2e = e2e_pageable = None
    if not args.no_e2e:
        fn = il.STRATEGIES[variant]
        # (--device-override: every rank on one GPU, so the list repeats it)
        e2e_devs = tuple(range(world)) if args.device_override is None else (args.device_override,) * world
        cfg_e2e = il.ExecConfig(mode=args.mode, devices=e2e_devs) if world > 1 else cfg
        host_group = None
        if dist is not None:
            torch.cuda.synchronize(dev)
            # the other ranks wait on a host-side (gloo) barrier: an NCCL
            # barrier would leave a spinning collective kernel on the very
            # GPUs rank 0's call is using
            host_group = dist.new_group(backend="gloo")
            dist.barrier(group=host_group)
        if rank == 0:
            # pinned host copies of the store buffers (inputs of every step)
            pinned = []
            for b in store.buffers:
                t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True)
                t.numpy()[:] = b
                pinned.append(t.numpy())
            hstore = il.LayoutStore(store.kind, store.precision, n, pinned, store.shapes)
            tq = torch.empty((m, 2), dtype=torch.float64, pin_memory=True)
            tq.numpy()[:] = queries
            hq = tq.numpy()  # pinned (m, 2) float64 queries
            pq = np.ascontiguousarray(queries)  # pageable
            pstore = il.LayoutStore(store.kind, store.precision, n,
                                    [np.array(b, copy=True) for b in store.buffers], store.shapes)

            def timed(st_, q_):
                for _ in range(min(args.warmup, 2)):
                    fn(st_, q_, params, cfg_e2e)
                t0 = time.perf_counter()
                for _ in range(args.steps):
                    res = fn(st_, q_, params, cfg_e2e)
                dt = time.perf_counter() - t0
                del res
                return dt

            t_e2e = timed(hstore, hq)
            # the same through the caller's plain (pageable) numpy buffers: the
            # reference's own run_* callers hold ordinary arrays
            t_pg = timed(pstore, pq)
            e = 4 if prec == "single" else 8
            # store buffers + the (m, 2) float64 query pairs (cast on the device, idw_run_xy)
            h2d = sum(b.nbytes for b in hstore.buffers) + 16 * m
            d2h = m * e
            api = (f"paper_1402_4986_b200.{fn.__name__}(LayoutStore[pinned host], queries[pinned host f64], "
                   f"Params(p={p}), ExecConfig(mode='{args.mode}'"
                   + (f", devices={e2e_devs}))" if world > 1 else "))"))
            e2e = {"value": total_pairs * args.steps / t_e2e / 1e9, "unit": "GPairs/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "api": api}
            e2e_pageable = {"value": total_pairs * args.steps / t_pg / 1e9, "unit": "GPairs/s",
                            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                            "api": api.replace("pinned host", "pageable host")}
        if dist is not None:
            dist.barrier(group=host_group)

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle

        threads = oracle.max_threads()
        v, msub, dt = cpu_sample(store, queries, p, args.cpu_seconds, threads)
        cpu = {"value": v, "unit": "GPairs/s", "cores": threads, "kind": "port",
               "sample": f"{n} data x {msub} queries ({dt:.1f} s), oracle/idw_oracle.c predict_block "
                         f"(reference kernels.py:34-67 restated in C), {threads} pthreads"}

    # ---- parity of the timed output (rank 0's shard; outside the timed region).
    # Each prediction depends only on its query and all n points
    # (kernels.py:42-67), so a strided query subsample checks it exactly.
    parity = None
    if rank == 0 and not args.no_parity:
        import numpy as np

        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle

        nchk = 1024 if n <= (1 << 20) else 256
        idx = np.unique(np.linspace(0, hi - lo - 1, nchk).astype(np.int64))
        got = out_l.cpu().numpy()[idx]
        sub = queries[lo:hi][idx]
        if args.mode == "fast":
            ref = oracle.truth(store, sub, p)
            kind = "oracle.truth (fp64 double-double on the run-precision inputs)"
        elif variant == "nested_improved":
            ref = oracle.nested_improved_mt(store, sub, p)
            kind = "oracle.nested_improved (reference nested_improved_block restated, G=1024)"
        else:
            ref = oracle.predict_mt(store, sub, p)
            kind = "oracle.predict (reference predict_block restated)"
        a, b = got.astype(np.float64), np.asarray(ref, np.float64)
        err = float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
        tol = 1e-5 if prec == "single" else 1e-12
        parity = {"max_rel_err": err, "queries_checked": int(idx.size), "oracle": kind,
                  "tolerance": tol, "pass": bool(err <= tol),
                  "bitwise": bool(np.array_equal(got, np.asarray(ref, got.dtype))) if args.mode == "exact" else None}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GPairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if prec == "single" else "f64",
            "data": "synthetic: splitmix64 uniform cloud (idwlayout generate_cloud_arrays, data seed 0, "
                    "query seed 1), x,y in [0,1), z in [0,100)",
            "config": {"workload": desc, "n": n, "m": m, "layout": layout, "precision": prec,
                       "variant": variant, "mode": args.mode, "p": p, "zero_eps": 0.0,
                       "parallelism": f"query-shard x{world} (data broadcast + gather per step)",
                       "l2": "flushed between steps (256 MiB write, outside the per-step event pairs); "
                             "inputs resident in HBM"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable,
            "clocks": clocks, "parity": parity,
            "gpu_launches": launches[0],
            "mufu_probe": {"rcp_per_s": probe_rate},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
