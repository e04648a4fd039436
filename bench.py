"""Benchmark: sampled edges/s (2-hop fanout 10, recent + uniform) and ingest edges/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config gdelt|reddit|wiki]

Workload (BASELINE.json metric, configs[3] at N GPUs; fits one B200):
GDELT-shaped synthetic stream -- 17,000 nodes, 191,000,000 directed edges,
tau 8192, power-law destinations and sources (skew 2.2), 175,200 time ticks
 -- drawn on the GPU with the reference generator's law
(paper_2311_17410_b200/synth.py), ingested in 100K-edge batches
through gf_graph_add_edges.  One step = sample_khop over R = 2^20 roots per
GPU (the last edges' src+dst at their own timestamps, harness.py:542-545)
with fanouts [10, 10], once with the recent and once with the uniform policy.
value = sampled edges (all hops, both policies, all ranks) / max-over-ranks
device time.  Multi-GPU: every rank holds a full replica (each new batch is
assembled with an NCCL all-gather of per-rank shards) and samples its own
2^20 roots with key base rank*2^20 (weak scaling, no data-path collective).

--impl reference times the reference algorithm on the host: the CPU oracle's
faithful restatement of sample_khop (oracle/gf_oracle.c, all host threads)
on a bounded root sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: nodes, edges, directed, tau, skew, src_skew, span, roots per GPU
    "gdelt": dict(nodes=17_000, edges=191_000_000, directed=True, tau=8192, skew=2.2, src_skew=2.2, span=175_200,
                  roots=1 << 20, label="GDELT-shaped TGN 2-hop f10 (17K nodes, 191M edges, directed, tau 8192)"),
    # configs[1]: TGAT uniform [10, 10]; roots = 2 x 600 per minibatch in the paper, 2^16 here to fill the GPU
    "reddit": dict(nodes=11_000, edges=672_000, directed=False, tau=48, skew=2.2, src_skew=None, span=2_592_000,
                   roots=1 << 16, policies=("uniform",),
                   label="REDDIT-shaped TGAT 2-hop f10 uniform (11K nodes, 672K edges, undirected, tau 48)"),
    # configs[0]: TGN recent [10] (the reference's CPU case); 8,000 roots = one 4,000-edge minibatch
    "wiki": dict(nodes=9_000, edges=157_000, directed=False, tau=48, skew=2.2, src_skew=None, span=2_592_000,
                 roots=8_000, fanouts=[10], policies=("recent",),
                 label="WIKI-shaped TGN 1-hop f10 recent (9K nodes, 157K edges, undirected, tau 48)"),
    # configs[4] at one GPU's share of the 8-way partition (owner = v % 8): 1/8 of the nodes and
    # edges of the MAG shape, GraphSAGE-temporal uniform [15, 10], 10M-edge ingest batches
    "mag8": dict(nodes=15_250_000, edges=162_500_000, directed=True, tau=8192, skew=2.2, src_skew=2.2, span=120,
                 roots=1 << 20, fanouts=[15, 10], policies=("uniform",), batch=10_000_000, blocks_per_node=4,
                 label="MAG-shaped 1/8 (one GPU's share of the 8-way partition: 15.25M nodes, 162.5M edges, "
                       "directed, tau 8192, span 120) GraphSAGE uniform [15,10]"),
}
FANOUTS = [10, 10]
POLICIES = ("recent", "uniform")
INGEST_BATCH = 100_000
# algorithmic bytes per query / per sampled edge
BYTES_PER_QUERY = 65
BYTES_PER_EDGE = 50


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """SM clock + throttle reasons sampled every 2 ms during the timed region (NVML in a thread;
    falls back to `nvidia-smi -lms 200` when NVML is unavailable)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.rows: list[tuple[float, float, list[str]]] = []
        self.stop = threading.Event()
        self.t = None
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.sample()  # at least one sample inside the region
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001 -- NVML missing: nvidia-smi below
            self.nv = None
        return self

    def sample(self):
        nv = self.nv
        mhz = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((mhz, self.max_mhz, [n for n, a in self.REASONS if mask & getattr(nv, a, 0)]))

    def _loop(self):
        while not self.stop.wait(0.002):
            try:
                self.sample()
            except Exception:  # noqa: BLE001
                return

    def __exit__(self, *exc):
        self.stop.set()
        if self.t is not None:
            self.t.join(timeout=2)
        if self.nv is not None:
            try:
                self.sample()
            except Exception:  # noqa: BLE001
                pass
        else:
            self._smi_once()

    def _smi_once(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True, timeout=10).stdout
            r = [x.strip() for x in out.split(",")]
            names = [n for n, _ in self.REASONS]
            self.rows.append((float(r[0]), float(r[1]), [n for n, v in zip(names, r[2:6]) if v.lower() == "active"]))
        except (OSError, ValueError, IndexError, subprocess.SubprocessError):
            pass

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.rows[0][1],
                "reasons": sorted({n for r in self.rows for n in r[2]}), "samples": len(self.rows),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


def self_launch(args) -> int | None:
    """--gpus N > 1 without a torchrun environment: re-run this command under torch.distributed.run
    with N ranks on 127.0.0.1 (one process per GPU) and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=dict(os.environ)).returncode


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        if args.gpus not in (1, world) and rank == 0:
            print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; running {world} ranks", file=sys.stderr)
        if _backend() == "gloo":
            # GF_BENCH_BACKEND=gloo: exercise the multi-rank path with several ranks sharing the GPUs
            # of a smaller box (ranks map to devices round-robin; host-staged collectives)
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            # the NCCL communicator-init lines (rank count, NVLink/NVLS transport) go to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            # failure propagation: the process group's watchdog polls
            # ncclCommGetAsyncError; on an asynchronous NCCL error or a collective past the timeout
            # it aborts the communicator and the waiting ranks raise instead of hanging
            os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                    timeout=datetime.timedelta(seconds=float(os.environ.get("GF_NCCL_TIMEOUT_S", "600"))))
        # one tiny collective so the communicator (and its INIT log) exists before any timing
        t = torch.ones(1, device=_coll_device())
        dist.all_reduce(t)
        if rank == 0:
            print(f"bench: {_backend()} communicator up, {int(t.item())} ranks", file=sys.stderr, flush=True)
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
    return world, rank, local


def _backend() -> str:
    return os.environ.get("GF_BENCH_BACKEND", "nccl")


def _coll_device() -> str:
    return "cpu" if _backend() == "gloo" else "cuda"


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_stream(cfg, device):
    from paper_2311_17410_b200.synth import generate_synthetic_device

    return generate_synthetic_device(cfg["nodes"], cfg["edges"], cfg["skew"], cfg["span"], seed=0,
                                     src_skew=cfg["src_skew"], device=device)


def roots_for_rank(src, dst, ts, R, rank):
    """Latest R/2 edges for this rank: src+dst at their own timestamps (harness.py:542-545)."""
    import torch

    half = R // 2
    e = src.numel()
    lo, hi = e - (rank + 1) * half, e - rank * half
    roots = torch.cat([src[lo:hi], dst[lo:hi]]).contiguous()
    rts = torch.cat([ts[lo:hi], ts[lo:hi]]).contiguous()
    return roots, rts


def build_graph(cfg, src, dst, ts, world, rank, device):
    """Ingest the stream in 100K-edge batches; N>1: each batch is all-gathered from per-rank shards.

    Warm-up (untimed): the first two batches go into a throwaway graph first, so the timed build does
    not carry the process's one-time costs (first cooperative launch, allocator segments for the
    per-batch outputs, NCCL's first all-gather)."""
    import torch

    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200.distributed import ReplicatedGraph, shard_range

    n = src.numel()

    def new_graph(edges):
        g = gf.DynamicGraph(directed=cfg["directed"], tau=cfg["tau"], device=device)
        slots = edges * (1 if cfg["directed"] else 2)
        g.reserve(cfg["nodes"], cfg["nodes"] * cfg.get("blocks_per_node", 16) + slots // max(1, cfg["tau"]) + 1024,
                  slots + min(cfg["nodes"] * cfg["tau"], slots // 2))
        return g

    def ingest(rg, lo, hi):
        # this rank's shard of the batch; N>1 all-gathers the shards (NCCL) before K1
        a, b = shard_range(hi - lo, world, rank)
        rg.ingest(src[lo + a:lo + b], dst[lo + a:lo + b], ts[lo + a:lo + b])

    warm_n = min(n, 2 * INGEST_BATCH)
    warm = ReplicatedGraph(new_graph(warm_n))
    for lo in range(0, warm_n, INGEST_BATCH):
        ingest(warm, lo, min(warm_n, lo + INGEST_BATCH))
    torch.cuda.synchronize()
    del warm
    g = new_graph(n)
    rg = ReplicatedGraph(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for lo in range(0, n, INGEST_BATCH):
        ingest(rg, lo, min(n, lo + INGEST_BATCH))
    e1.record()
    torch.cuda.synchronize()
    return g, e0.elapsed_time(e1)


def replay_roots_for_rank(src, dst, ts, R, rank):
    """Replay roots: R/2 edges drawn uniformly (seed 1 + rank) from the whole
    stream, src+dst at their own timestamps -- deep boundaries, as in harness.py:383-389."""
    import torch

    gen = torch.Generator(device=src.device)
    gen.manual_seed(1 + rank)
    idx = torch.randint(0, src.numel(), (R // 2,), generator=gen, device=src.device)
    return torch.cat([src[idx], dst[idx]]).contiguous(), torch.cat([ts[idx], ts[idx]]).contiguous()


def timed_steps(g, roots, rts, key_base, steps, policies=None):
    """Device time (ms, CUDA events on the current stream) and sampled edges of `steps` steps."""
    import torch

    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run_step(g, roots, rts, key_base, policies)
    torch.cuda.synchronize()
    a.record(stream)
    edges = 0
    for _ in range(steps):
        edges += run_step(g, roots, rts, key_base, policies)[0]
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b), edges


def run_step(g, roots, rts, R_base, policies=None):
    import paper_2311_17410_b200 as gf

    edges = 0
    queries = 0
    out = []
    for pol in policies or POLICIES:
        s = gf.sample_khop_device(g, roots, rts, FANOUTS, gf.SamplingPolicy(pol), seed=0, root_key_base=R_base)
        for lay in s.layers:
            edges += int(lay.neighbors.numel())
            queries += int(lay.source_nodes.numel())
        out.append(s)
    return edges, queries, out


def cpu_oracle_graph(cfg, src, dst, ts):
    """Build the oracle (reference restatement) graph on the host; returns (graph, ingest edges/s)."""
    from oracle import OracleGraph

    s, d, t = src.cpu().numpy(), dst.cpu().numpy(), ts.cpu().numpy()
    o = OracleGraph(cfg["directed"], cfg["tau"])
    t0 = time.perf_counter()
    for lo in range(0, len(s), INGEST_BATCH):
        o.add_edges(s[lo:lo + INGEST_BATCH], d[lo:lo + INGEST_BATCH], t[lo:lo + INGEST_BATCH])
    return o, len(s) / (time.perf_counter() - t0)


def cpu_sample_rate(o, roots, rts, faithful: bool, budget_s: float, chunk: int, threads: int):
    """Time the oracle's sample_khop (recent + uniform) over successive root chunks until budget_s."""
    edges, used, t_total = 0, 0, 0.0
    pos = 0
    while t_total < budget_s and pos < len(roots):
        r, t = roots[pos:pos + chunk], rts[pos:pos + chunk]
        t0 = time.perf_counter()
        for pol in POLICIES:
            lays = o.sample_khop(r, t, FANOUTS, pol, seed=0, root_key_base=pos, threads=threads, faithful=faithful)
            edges += sum(len(lay[3]) for lay in lays)
        t_total += time.perf_counter() - t0
        used += len(r)
        pos += chunk
    return edges / t_total if t_total else 0.0, used, edges, t_total


TRAFFIC_SOURCES = ("bench.py", "paper_2311_17410_b200/csrc/gf_sample.cu", "paper_2311_17410_b200/csrc/gf_graph.cuh")
# profiles/r01_randread.md: one random 32 B record costs a 128 B line; ~37.5 G lines/s on a B200
RANDOM_LINE_CAP = {"lines_per_s": 37.5e9, "bytes_per_line": 128, "source": "profiles/r01_randread.md"}


def source_sha16() -> str:
    """Hash of the files whose change invalidates an ncu traffic capture (scripts/ncu_summarize.py)."""
    import hashlib

    h = hashlib.sha256()
    for f in TRAFFIC_SOURCES:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def load_traffic() -> dict:
    """profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per sampler launch
    from one ncu capture of this workload (scripts/ncu_sampler.sh + scripts/ncu_summarize.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def launch_key(name: str) -> str:
    """'k_sample_fused<false>[uniform/hop1]' -> 'k_sample_fused[uniform/hop1]'."""
    return re.sub(r"<.*?>|\(\)", "", name)


def bench_ours(args, cfg, world, rank, local):
    import gc

    import torch

    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200 import _lib

    # as timeit does: no collector pauses inside timed regions (every sampling / ingest / fetch call
    # synchronises with the host once, so a pause would show up as device idle time; single fetch
    # passes measured up to 5x slower with the collector on)
    gc.collect()
    gc.disable()
    device = torch.device("cuda", local)
    R = cfg["roots"] if args.roots is None else args.roots
    if args.strong:  # fixed total root count (R = 2^23 split over the ranks)
        R = max(2, (args.strong // world) // 2 * 2)
    src, dst, ts = make_stream(cfg, device)
    torch.cuda.synchronize()
    g, ingest_ms = build_graph(cfg, src, dst, ts, world, rank, device)
    deleted = None
    if args.deleted:
        # the general (post-deletion) sampler: soft-delete 1% of the edges (storage.py:479-505); every
        # later call scans candidate validity (sampling.py:178) instead of the fused fast path
        gen = torch.Generator(device=device)
        gen.manual_seed(3)
        ids = torch.randperm(src.numel(), generator=gen, device=device)[: src.numel() // 100].sort().values
        deleted = {"edges": int(g.delete_edges(ids)), "sampler": "post-deletion path: k_sample_fused_del (lane per query, validity-checked selection)"}
    roots, rts = roots_for_rank(src, dst, ts, R, rank)
    key_base = rank * R

    for _ in range(args.warmup):
        run_step(g, roots, rts, key_base)
    torch.cuda.synchronize()
    barrier(world)
    launches0 = _lib.launch_count()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    edges = queries = 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            e, q, _ = run_step(g, roots, rts, key_base)
            edges += e
            queries += q
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms_local = ev0.elapsed_time(ev1)
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(ms_local, world)
    total_edges = sum_over_ranks(edges, world)
    value = total_edges / (ms / 1e3)

    # per-kernel shares (separate profiled pass, same workload)
    _lib.profile_enable(True)
    e_p, q_p, outs_p = run_step(g, roots, rts, key_base)
    prof = _lib.profile_summary()
    _lib.profile_enable(False)
    # per (policy, hop) layer sizes for the per-launch algorithmic bytes:
    # count kernel 65 B/query, write kernel 50 B/sampled edge
    layer_qs = {}
    for pol, s_ in zip(POLICIES, outs_p):
        for h, lay in enumerate(s_.layers):
            layer_qs[f"{pol}/hop{h}"] = (int(lay.source_nodes.numel()), int(lay.neighbors.numel()))
    pk = peaks()
    kernels, base_ms, base_bytes = {}, {}, {}
    tot_ms = sum(v[1] for v in prof.values())
    for name, (cnt, kms) in sorted(prof.items()):
        raw = name.split("[")[0]
        tag = name[len(raw) + 1:-1] if "[" in name else None
        base = re.sub(r"[()]|<.*>", "", raw).strip()
        ent = {"launches": cnt, "ms": round(kms, 4), "share": round(kms / tot_ms, 4) if tot_ms else None}
        if tag in layer_qs and base.startswith(("k_count", "k_write", "k_sample_fused")):
            q_l, s_l = layer_qs[tag]
            b = (BYTES_PER_QUERY * q_l if base.startswith("k_count") else
                 BYTES_PER_EDGE * s_l if base.startswith("k_write") else BYTES_PER_QUERY * q_l + BYTES_PER_EDGE * s_l)
            ent["alg_bytes"] = b
            ent["achieved_gbs"] = round(b / (kms / 1e3) / 1e9, 1) if kms > 0 else None
            base_bytes[base] = base_bytes.get(base, 0) + b
        base_ms[base] = base_ms.get(base, 0.0) + kms
        kernels[name] = ent
    for ent in kernels.values():
        if ent.get("achieved_gbs"):
            ent["frac"] = round(ent["achieved_gbs"] / pk["hbm_gbs"], 4)
    dom_name = max(base_bytes, key=lambda k: base_ms[k])
    achieved = base_bytes[dom_name] / (base_ms[dom_name] / 1e3) / 1e9
    # the dominant single launch and its measured DRAM traffic (ncu capture of this config, keyed by
    # the hash of the sources it depends on)
    dom_launch = max((k for k in kernels if "alg_bytes" in kernels[k]), key=lambda k: kernels[k]["ms"])
    tr = load_traffic()
    sha = source_sha16()
    tr_launch = (tr.get("launches") or {}).get(launch_key(dom_launch)) if tr.get("config") == args.config else None
    traffic = tr_launch["dram_bytes"] if tr_launch else None
    dom = {"launch": dom_launch, "ms": kernels[dom_launch]["ms"], "alg_bytes": kernels[dom_launch]["alg_bytes"],
           "achieved_gbs": kernels[dom_launch]["achieved_gbs"], "frac": kernels[dom_launch]["frac"],
           "traffic": traffic, "traffic_ratio": round(traffic / kernels[dom_launch]["alg_bytes"], 3) if traffic else None,
           "traffic_source": "profiles/ncu_traffic.json" if traffic else None,
           "traffic_sha_match": (tr.get("source_sha16") == sha) if traffic else None}
    if traffic:
        dom["ncu_ms"] = tr_launch.get("ms")
    pipe_ms = sum(v for k, v in base_ms.items() if k.startswith(("k_count", "k_write", "k_total", "cub_scan", "k_sample_fused")))
    pipe_gbs = (BYTES_PER_QUERY * q_p + BYTES_PER_EDGE * e_p) / (pipe_ms / 1e3) / 1e9 if pipe_ms else None

    # e2e through the public API with host (pinned) buffers: H2D roots, sample, D2H every layer
    e2e = None
    if not args.no_e2e:
        roots_h = roots.cpu().pin_memory()
        rts_h = rts.cpu().pin_memory()
        _, _, outs = run_step(g, roots, rts, key_base)
        host_bufs = []
        bo = 0
        for s in outs:
            for lay in s.layers:
                for t in (lay.offsets, lay.neighbors, lay.edge_ids, lay.timestamps):
                    host_bufs.append(torch.empty(t.numel() + (1 << 20), dtype=torch.int64).pin_memory())
        sampler = {p: gf.TemporalSampler(g, FANOUTS, p, seed=0) for p in POLICIES}
        torch.cuda.synchronize()
        barrier(world)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_edges = 0
        # results go back on a copy stream, so one policy's D2H overlaps the next policy's sampling
        # (the D2H over PCIe is ~20x the sampling time)
        copy_stream = torch.cuda.Stream(device=device)
        a0.record(stream)
        for _ in range(args.steps):
            bi = bo = 0
            k = 0
            for p in POLICIES:
                r_d = roots_h.to(device, non_blocking=True)
                t_d = rts_h.to(device, non_blocking=True)
                bi += 2 * roots_h.numel() * 8
                s = sampler[p].sample(r_d, t_d, root_key_base=key_base)
                copy_stream.wait_stream(stream)
                with torch.cuda.stream(copy_stream):
                    for lay in s.layers:
                        e2e_edges += int(lay.neighbors.numel())
                        for t in (lay.offsets, lay.neighbors, lay.edge_ids, lay.timestamps):
                            t.record_stream(copy_stream)  # the allocator keeps it until the copy is done
                            hb = host_bufs[k]
                            k += 1
                            hb[: t.numel()].copy_(t, non_blocking=True)
                            bo += t.numel() * 8
        stream.wait_stream(copy_stream)
        a1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        e2e_ms = max_over_ranks(a0.elapsed_time(a1), world)
        e2e_total = sum_over_ranks(e2e_edges, world)
        e2e = {"value": round(e2e_total / (e2e_ms / 1e3), 1), "unit": "sampled edges/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo}

    # secondary numbers (rank-local, not the headline): each policy alone, and the replay root set
    per_policy = {}
    for pol in POLICIES:
        pms, pe = timed_steps(g, roots, rts, key_base, 3, (pol,))
        qs = [v for k_, v in layer_qs.items() if k_.startswith(pol + "/")]
        pb = sum(BYTES_PER_QUERY * q_ + BYTES_PER_EDGE * s_ for q_, s_ in qs)
        per_policy[pol] = {"value": round(pe / (pms / 1e3), 1), "ms_per_step": round(pms / 3, 4),
                           "alg_bytes_per_step": pb,
                           "frac": round(pb / (pms / 3 / 1e3) / 1e9 / pk["hbm_gbs"], 4)}
        if pol == "uniform":
            # every uniform pick is one random record: at most RANDOM_LINE_CAP lines/s, so the policy's
            # algorithmic fraction cannot exceed (picks/s at the cap) * alg bytes per pick / peak
            s_tot = sum(s_ for _, s_ in qs)
            cap_ms = s_tot / RANDOM_LINE_CAP["lines_per_s"] * 1e3
            per_policy[pol]["random_line_cap"] = {**RANDOM_LINE_CAP, "picks_per_step": s_tot,
                                                  "floor_ms_per_step": round(cap_ms, 4),
                                                  "frac_cap": round(pb / (cap_ms / 1e3) / 1e9 / pk["hbm_gbs"], 4)}
    rroots, rrts = replay_roots_for_rank(src, dst, ts, R, rank)
    rms, re_ = timed_steps(g, rroots, rrts, key_base, 3)
    replay = {"value": round(re_ / (rms / 1e3), 1), "unit": "sampled edges/s", "ms_per_step": round(rms / 3, 4),
              "roots": "R/2 uniformly drawn edges (seed 1+rank), src+dst at own ts (SURVEY.md 8(d)(ii))"}
    del rroots, rrts

    fetch = fetch_bench(g, src, dst, ts, cfg, device, world=world, rank=rank) \
        if (args.config == "gdelt" and not args.no_fetch) else None

    ingest_eps = cfg["edges"] / (max_over_ranks(ingest_ms, world) / 1e3)
    info = g.info()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, src, dst, ts, roots, rts, args)

    if rank == 0:
        line = {
            "metric": "sampled edges/sec (2-hop fanout 10, recent+uniform) at 1/2/4/8 B200; edges/sec ingest",
            "value": round(value, 1),
            "unit": "sampled edges/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None,
            "dtype": "int64",
            "data": "synthetic (reference generator law, drawn on device; seed 0)",
            "config": {
                "workload": cfg["label"],
                "nodes": cfg["nodes"], "edges": cfg["edges"], "directed": cfg["directed"], "tau": cfg["tau"],
                "fanouts": FANOUTS, "policies": list(POLICIES), "roots_per_gpu": R,
                "roots": "latest R/2 edges per rank, src+dst at own ts (harness.py:542-545)",
                "ingest_batch": INGEST_BATCH,
                "l2": "no flush: slot pool %.1f GB >> 126 MB L2" % (info.slots_allocated * 32 / 1e9),
                "parallelism": f"replicas x{world}, root sharding (dp{world})",
            },
            "ingest": {"value": round(ingest_eps, 1), "unit": "edges/s",
                       "note": f"{INGEST_BATCH // 1000}K-edge batches through gf_graph_add_edges, device events over the whole build after an untimed 2-batch warm-up into a throwaway graph; N>1 includes the NCCL all-gather"},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 1), "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
                         "peak_source": pk["source"],
                         "alg_bytes": f"{BYTES_PER_QUERY} B/query + {BYTES_PER_EDGE} B/sampled edge (SURVEY.md 8(d)); fused kernel = both",
                         "pipeline_gbs": round(pipe_gbs, 1) if pipe_gbs else None,
                         "pipeline_frac": round(pipe_gbs / pk["hbm_gbs"], 4) if pipe_gbs else None,
                         "dominant_launch": dom, "source_sha16": sha,
                         **(l2_fraction(cfg, info, base_bytes[dom_name], base_ms[dom_name]) or {})},
            "kernels": kernels,
            "per_policy": per_policy,
            "fetch": fetch,
            "replay": replay,
            "deleted": deleted,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def l2_fraction(cfg, info, alg_bytes, ms) -> dict | None:
    """Stores that fit the 126 MB L2 (WIKI/REDDIT shapes) are bound by L2, not HBM, bandwidth: report
    the kernel's algorithmic bytes against the measured L2 read bandwidth (profiles/l2_bandwidth.json,
    scripts/l2bw.cu) next to the HBM fraction."""
    # the sampler's working set: 32 B slot records + the int32 timestamp copy + 128 B node records
    store_bytes = info.slots_allocated * 36 + info.num_nodes * 128
    if store_bytes > 126e6:
        return None
    p = os.path.join(ROOT, "profiles", "l2_bandwidth.json")
    if not os.path.exists(p):
        return {"l2_resident_store_bytes": store_bytes, "l2_peak_gbs": None}
    with open(p) as fh:
        l2 = json.load(fh)
    gbs = alg_bytes / (ms / 1e3) / 1e9
    return {"l2_resident_store_bytes": store_bytes, "l2_peak_gbs": l2["l2_read_gbs"],
            "l2_frac": round(gbs / l2["l2_read_gbs"], 4), "l2_source": "profiles/l2_bandwidth.json"}


# GDELT feature dims and cache sizes (3% of nodes / 3 per mille of edges)
FETCH_DV, FETCH_DE = 413, 186
FETCH_MINIBATCH = 4000      # TGN minibatch edges -> 8,000 roots (harness.py:424-429)
FETCH_EDGE_TABLE = 5_000_000  # edge features held for the latest 5M edges (142 GB for all 191M)


def fetch_bench(g, src, dst, ts, cfg, device, batches: int = 50, world: int = 1, rank: int = 0) -> dict:
    """Feature-cache fetch block (harness.py:432-446) on GPU: per minibatch of the latest edges,
    2-hop recent f10 sample, then node keys = roots + last-layer neighbours through an LRU node cache
    (d_v 413) and edge keys = every layer's edge ids through an LRU edge cache (d_e 186); misses
    are filled from the device feature tables and inserted.  Unit: one fetched row
    (8 B key + 1 B mask + 8*d B read+write)."""
    import torch

    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200 import _lib

    nodes = cfg["nodes"]
    gen = torch.Generator(device=device)
    gen.manual_seed(7)
    ntab = gf.NodeFeatureTable(FETCH_DV, device=device)
    ntab.set_many(torch.arange(nodes, device=device), torch.rand(nodes, FETCH_DV, device=device, generator=gen))
    e_total = src.numel()
    e0 = e_total - FETCH_EDGE_TABLE
    etab = gf.EdgeFeatureTable(FETCH_DE, device=device)
    # N > 1: edge rows sharded by eid % N (each rank stores its share; misses are fetched from the
    # owners over NCCL inside the fetch block); node rows are small and replicated
    from paper_2311_17410_b200.distributed import ShardedFeatureTable, fetch_features_sharded

    eids = torch.arange(e0, e_total, device=device)
    erows = torch.rand(FETCH_EDGE_TABLE, FETCH_DE, device=device, generator=gen)
    own = ShardedFeatureTable.owns(eids, world, rank)
    etab.append(eids[own].contiguous(), erows[own].contiguous())
    del erows
    eshard = ShardedFeatureTable(etab)
    ncache = gf.VectorCache("lru", max(1, int(0.03 * nodes)), FETCH_DV, 0.2, device=device)
    ecache = gf.VectorCache("lru", max(1, int(0.003 * e_total)), FETCH_DE, 0.2, device=device)
    mb = []
    for b in range(batches + 2):  # minibatches walking back from the newest edges
        hi = e_total - b * FETCH_MINIBATCH
        lo = hi - FETCH_MINIBATCH
        roots = torch.cat([src[lo:hi], dst[lo:hi]]).contiguous()
        rts = torch.cat([ts[lo:hi], ts[lo:hi]]).contiguous()
        smp = gf.sample_khop_device(g, roots, rts, FANOUTS, gf.SamplingPolicy("recent"), seed=0)
        nkeys = torch.cat([roots, smp.layers[-1].neighbors]).contiguous()
        ekeys = torch.cat([lay.edge_ids for lay in smp.layers]).contiguous()
        mb.append((nkeys, ekeys))
    # reserve the largest output blocks once, so the caching allocator never grows inside the timed loop
    mx_n, mx_e = max(int(nk.numel()) for nk, _ in mb), max(int(ek.numel()) for _, ek in mb)
    held = [torch.empty((mx_n, FETCH_DV), dtype=torch.float32, device=device),
            torch.empty((mx_e, FETCH_DE), dtype=torch.float32, device=device)]
    del held
    for nk, ek in mb[:2]:  # warm-up
        gf.fetch_features(ncache, ntab, nk)
        fetch_features_sharded(ecache, eshard, ek)
    torch.cuda.synchronize()
    # every pass starts from the same post-warm-up cache state (device snapshots), so passes 2 and
    # 3 replay the streaming minibatches of pass 1 rather than a cache they already warmed
    nsnap, esnap = ncache.device_snapshot(), ecache.device_snapshot()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rows = sum(nk.numel() + ek.numel() for nk, ek in mb[2:])
    byts = sum(nk.numel() * (9 + 8 * FETCH_DV) + ek.numel() * (9 + 8 * FETCH_DE) for nk, ek in mb[2:])
    passes, hit_rates = [], []
    diag = os.environ.get("GF_FETCH_DIAG") is not None  # per-call host times to stderr (diagnostics only)
    diag_rows = []
    for _ in range(5):
        nsnap.restore_into(ncache)
        esnap.restore_into(ecache)
        ncache.reset_stats()
        ecache.reset_stats()
        torch.cuda.synchronize()
        a.record()
        for nk, ek in mb[2:]:
            t0 = time.perf_counter() if diag else 0.0
            gf.fetch_features(ncache, ntab, nk)
            t1 = time.perf_counter() if diag else 0.0
            fetch_features_sharded(ecache, eshard, ek)
            if diag:
                t2 = time.perf_counter()
                diag_rows.append((round((t1 - t0) * 1e3, 3), round((t2 - t1) * 1e3, 3)))
        b.record()
        torch.cuda.synchronize()
        passes.append(a.elapsed_time(b))
        hit_rates.append((ncache.stats()["hit_rate"], ecache.stats()["hit_rate"]))
    ms = statistics.median(passes)
    if diag:
        worst = sorted(range(len(diag_rows)), key=lambda i: -sum(diag_rows[i]))[:8]
        print("fetch diag: passes", passes, "slowest calls (index, node ms, edge ms):",
              [(i, diag_rows[i]) for i in worst], file=sys.stderr)
    _lib.profile_enable(True)
    for nk, ek in mb[2:6]:
        gf.fetch_features(ncache, ntab, nk)
        fetch_features_sharded(ecache, eshard, ek)
    prof = _lib.profile_summary()
    _lib.profile_enable(False)
    tot = sum(v[1] for v in prof.values())
    gat = sum(v[1] for k, v in prof.items() if k.startswith(("k_gather_rows", "k_fetch_gather", "k_fill_from_table",
                                                                  "k_copy_rows")))
    pk = peaks()
    gbs = byts / (ms / 1e3) / 1e9
    return {"value": round(rows / (ms / 1e3), 1), "unit": "fetched rows/s", "ms_per_minibatch": round(ms / batches, 4),
            "rows_per_minibatch": rows // batches, "achieved_gbs": round(gbs, 1), "frac": round(gbs / pk["hbm_gbs"], 4),
            "row_copy_share": round(gat / tot, 3) if tot else None,
            "passes_ms": [round(x, 3) for x in passes],
            "pass1_rows_per_s": round(rows / (passes[0] / 1e3), 1),
            "edge_rows": f"sharded by eid % {world} over the ranks (misses fetched from the owners)" if world > 1
                         else "local table",
            "top_kernels": {k: round(v[1] / tot, 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]},
            "node_hit_rate": round(hit_rates[0][0], 4), "edge_hit_rate": round(hit_rates[0][1], 4),
            "config": f"GDELT TGN minibatch {FETCH_MINIBATCH} edges -> {2 * FETCH_MINIBATCH} roots, 2-hop recent f10; "
                      f"node LRU cache 3% (d_v {FETCH_DV}), edge LRU cache 3 per mille (d_e {FETCH_DE}); "
                      f"edge table = latest {FETCH_EDGE_TABLE // 1_000_000}M edges; median of 5 passes over {batches} "
                      f"minibatches, each pass from the same restored post-warm-up caches"}


def cpu_baseline(cfg, src, dst, ts, roots, rts, args):
    threads = os.cpu_count() or 1
    o, cpu_ingest = cpu_oracle_graph(cfg, src, dst, ts)
    r, t = roots.cpu().numpy(), rts.cpu().numpy()
    rate, used, edges, secs = cpu_sample_rate(o, r, t, True, args.cpu_budget, 16, threads)
    frate, fused, fedges, fsecs = cpu_sample_rate(o, r, t, False, min(5.0, args.cpu_budget), 2048, threads)
    return {"value": round(rate, 1), "unit": "sampled edges/s", "cores": threads, "kind": "port",
            "sample": f"faithful C restatement of the reference sample_khop (candidate collection as "
                      f"sampling.py:145-182) on the same graph: first {used} of the {len(r)} roots, recent+uniform "
                      f"2-hop f10, {edges} edges in {secs:.1f}s",
            "ingest_edges_per_s": round(cpu_ingest, 1),
            "ingest_note": "oracle add_edges, 1 core (the reference add_edges is a serial loop)",
            "fast_port": {"value": round(frate, 1), "cores": threads,
                          "sample": f"early-exit C port (same output): {fused} roots, {fedges} edges in {fsecs:.1f}s"}}


def bench_reference(args, cfg, world, rank, local):
    """--impl reference: the reference algorithm (faithful oracle port) on host cores, rank 0 only."""
    if rank != 0:
        return
    import torch

    device = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    src, dst, ts = make_stream(cfg, device)
    R = cfg["roots"] if args.roots is None else args.roots
    roots, rts = roots_for_rank(src, dst, ts, R, 0)
    o, cpu_ingest = cpu_oracle_graph(cfg, src, dst, ts)
    r, t = roots.cpu().numpy(), rts.cpu().numpy()
    threads = os.cpu_count() or 1
    chunk = args.ref_chunk
    pos = 0
    for _ in range(args.warmup):
        cpu_sample_rate(o, r[pos:pos + chunk], t[pos:pos + chunk], True, 1e9, chunk, threads)
        pos += chunk
    edges, secs = 0, 0.0
    for _ in range(args.steps):
        _, _, e, s = cpu_sample_rate(o, r[pos:pos + chunk], t[pos:pos + chunk], True, 1e9, chunk, threads)
        edges += e
        secs += s
        pos += chunk
    value = edges / secs if secs else 0.0
    line = {
        "impl": "reference",
        "metric": "sampled edges/sec (2-hop fanout 10, recent+uniform) at 1/2/4/8 B200; edges/sec ingest",
        "value": round(value, 1), "unit": "sampled edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(secs * 1e3 / max(args.steps, 1), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic (same stream as --impl ours)",
        "config": {"workload": cfg["label"], "fanouts": FANOUTS, "policies": list(POLICIES), "roots_per_step": chunk,
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": round(value, 1), "unit": "sampled edges/s", "cores": threads, "kind": "port",
                         "sample": f"{chunk} roots per step of the same root set, faithful restatement of the "
                                   f"reference sample_khop (oracle/gf_oracle.c)"},
        "ingest": {"value": round(cpu_ingest, 1), "unit": "edges/s", "note": "oracle add_edges, 1 core"},
        "e2e": {"value": round(value, 1), "unit": "sampled edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="gdelt")
    ap.add_argument("--roots", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fetch", action="store_true")
    ap.add_argument("--strong", type=int, default=0, metavar="TOTAL_ROOTS",
                    help="strong scaling: TOTAL_ROOTS split over the ranks (default: 2^20 roots per rank, weak)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--deleted", action="store_true", help="soft-delete 1%% of the edges first (general sampler path)")
    ap.add_argument("--ref-chunk", type=int, default=16)
    args = ap.parse_args()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    cfg = CONFIGS[args.config]
    global FANOUTS, POLICIES, INGEST_BATCH
    FANOUTS = list(cfg.get("fanouts", FANOUTS))
    POLICIES = tuple(cfg.get("policies", POLICIES))
    INGEST_BATCH = cfg.get("batch", INGEST_BATCH)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        bench_reference(args, cfg, world, rank, local)
    else:
        bench_ours(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
