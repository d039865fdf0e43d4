#!/usr/bin/env python
"""Benchmark of the sparse gated-FFN forward (TwELL) on B200 — prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7B] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself through torch.distributed.run (one process per GPU,
rendezvous on 127.0.0.1); only rank 0 prints.

A step = one pass of the whole hot path (pack: gate GEMM -> TwELL, then the fused sparse up/down; plus
the NCCL all-reduce of partial outputs when N > 1) over one batch of M synthetic tokens, inputs and
weights resident in HBM.  The L2 is flushed (a 512 MiB write) between timed steps; every step is timed
with CUDA events on the launching stream; the reported time is the max over ranks.

N > 1 (torchrun): hidden-dim sharding (north_star (5)) — rank r owns N/G hidden units of all three weights
(contiguous rows, or TwELL tiles dealt round-robin with --shard-mode round_robin); every rank sees all M tokens;
value = M / t, the whole job's tokens/s (strong scaling: total work fixed); tokens_per_s_per_gpu = value / N is the
metric's per-GPU figure.

--impl reference: the CPU oracle (oracle/, plain fp64 C) timed on this box's host cores, on a bounded
row sample of the same workload per step (the only other place bench.py executes oracle/ besides the
cpu_baseline leg).  Rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "sparse-FFN fwd tokens/s/GPU @99% sparsity; speedup vs own dense FFN; HBM %"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}
FMA_LANES_PER_SM = 128
N_SMS = 148
# per-SM L2->SM ingress ceiling measured on this pool's B200s with the feed microbenchmark (tools/exp_feed.cu,
# profiles/r02/exp_feed_grid.txt: TMA tiles + cp.async gathers saturate at ~58 B/cycle/SM at 148, 74 and 37 SMs) —
# the binding limit of the union GEMMs (DESIGN.md §7 "Per-SM feed limits")
INGRESS_B_PER_CYCLE_SM = 58.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback (B200_PROFILING.md)"
    return d


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(argv, n: int) -> int:
    """--gpus N > 1 outside torchrun: one process per GPU through torch.distributed.run, rendezvous on 127.0.0.1
    (the driver's own launch form); rank 0's JSON line reaches our stdout, the exit code is propagated."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ, SFFN_BENCH_LAUNCHED="1")
    return subprocess.run(cmd, env=env).returncode


def bench_config(cfg, args, world: int) -> dict:
    """The `config` object of the JSON line — a function of the arguments only, so the reference arm and this arm
    print identical objects for the same command line."""
    replicas = world > 1 and args.shard == "tokens"
    par = "single" if world == 1 else (f"token replicas x{world}" if replicas else
                                       f"hidden-dim x{world} ({args.shard_mode})")
    return {"workload": cfg.name, "M": cfg.M, "K": cfg.K, "N": cfg.N, "T": cfg.T, "C": cfg.C, "sparsity": cfg.sparsity,
            "parallelism": par, "allreduce": "none" if world == 1 or replicas else args.allreduce,
            "l2": "flushed (512 MiB write) between timed steps", "seed": cfg.seed,
            "launch": "eager" if (args.no_graph or world > 1) else "cuda_graph"}


# ----------------------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a few hundred ms to start sampling: wait for its first line so that even a short
            # timed region (a few steps) is covered
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.n0 = len(self.lines)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        t0 = time.time()
        while len(self.lines) <= getattr(self, "n0", 0) and time.time() - t0 < 2.0:
            time.sleep(0.01)  # at least one sample taken after the region started
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle timing
def time_oracle(cfg, rows: int, p=None, kind: str = "sparse"):
    """The oracle as it stands on `rows` contiguous token rows.  kind="sparse": its TwELL-based forward (fp64 gate
    GEMM + Alg.1 pack + Eq.3 over the stored entries, SPEC's CPU criterion S:728); kind="dense": dense Eq.1 (fp64,
    3 M K N MACs) + the explicit TwELL pack."""
    import oracle
    X = synth.gen_x(cfg, 0, rows, p=p)
    Wg, Wu, Wd = synth.gen_w(cfg, "g"), synth.gen_w(cfg, "u"), synth.gen_w(cfg, "d")
    t0 = time.perf_counter()
    words, counts, ov, A = oracle.pack_from_inputs(X, Wg, cfg.T, cfg.C)
    if kind == "sparse":
        oracle.ffn_twell(X, words, Wu, Wd, cfg.N, cfg.T, cfg.C)
    else:
        oracle.ffn_dense(X, Wg, Wu, Wd)
    return time.perf_counter() - t0


def oracle_threads() -> int:
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n and n.isdigit() else (os.cpu_count() or 1)


def oracle_sample_rows(cfg, target_s: float = 15.0, kind: str = "sparse"):
    """Rows of CPU work of about target_s seconds: calibrate on a few rows, then scale (rows are independent).
    Rows are a multiple of the thread count (OpenMP over rows) so every core has work."""
    ncpu = oracle_threads()
    r0 = max(1, min(ncpu, 8))
    t = time_oracle(cfg, r0, kind=kind)
    rows = int(max(r0, min(cfg.M, r0 * target_s / max(t, 1e-3))))
    rows = max(r0, (rows // ncpu) * ncpu) if rows >= ncpu else rows
    return rows, t, r0


def cpu_baseline_leg(cfg, p, target_s: float) -> dict:
    """cpu_baseline: the oracle's sparse forward (the reported value) and its dense Eq.1 + pack,
    each on a bounded contiguous row sample, on this box's host cores."""
    ncpu = oracle_threads()
    rows, _, _ = oracle_sample_rows(cfg, target_s=target_s)
    t_o = time_oracle(cfg, rows, p)
    rows_d, _, _ = oracle_sample_rows(cfg, target_s=target_s / 2, kind="dense")
    t_d = time_oracle(cfg, rows_d, p, kind="dense")
    return {"value": rows / t_o, "unit": "tokens/s", "cores": min(ncpu, rows), "kind": "oracle",
            "cpu_model": cpu_model(), "omp_threads": ncpu,
            "sample": f"{rows} contiguous token rows of {cfg.name} (M={cfg.M}): fp64 gate GEMM + Alg.1 pack + Eq.3 over "
                      f"the stored entries ({t_o:.1f} s)",
            "dense_eq1_pack": {"value": rows_d / t_d, "unit": "tokens/s", "cores": min(ncpu, rows_d),
                               "sample": f"{rows_d} contiguous token rows: fp64 dense Eq.1 (3 M K N MACs) + the "
                                         f"TwELL pack ({t_d:.1f} s)"}}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle, each step a bounded row sample of the workload (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if "LOCAL_RANK" in os.environ:
        # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 is the only worker here, so it takes every host core
        # (read by the oracle's OpenMP runtime when oracle/ is first loaded, below)
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    ncpu = oracle_threads()
    p = synth.token_targets(cfg)
    # one step ~ a few seconds of oracle work so the whole run stays within minutes
    rows, t_cal, r_cal = oracle_sample_rows(cfg, target_s=max(1.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        time_oracle(cfg, rows, p)
    times = [time_oracle(cfg, rows, p) for _ in range(args.steps)]
    t = float(np.mean(times))
    val = rows / t
    sample = (f"{rows} contiguous token rows of {cfg.name} (M={cfg.M}) per step; fp64 gate GEMM + Alg.1 pack + Eq.3 "
              f"over the stored entries")
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    out = {"metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
           "scaling": "strong" if world > 1 and args.shard == "hidden" else "weak", "vs_baseline": None,
           "dtype": "f64", "data": DATA, "config": bench_config(cfg, args, world), "impl": "reference",
           "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": min(ncpu, rows), "kind": "oracle",
                            "sample": sample, "cpu_model": cpu_model(), "omp_threads": ncpu},
           "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


DATA = ("synthetic (seeded dyadic-grid generator: 99% sparsity, lognormal per-token nnz, lognormal per-neuron "
        "popularity, 30% dead neurons)")


def run_dry(args, cfg):
    """--dry-run (CPU, gloo): the multi-rank skeleton of this script without a GPU — rendezvous, this rank's hidden
    shard, max-over-ranks of a per-rank number, rank 0 prints one JSON line.  tests/test_bench_launch.py runs it
    through the self-launcher."""
    import torch
    import torch.distributed as dist

    from paper_2603_23198_b200.sharding import shard_perm, shard_range
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    n0, Nl = shard_range(cfg.N, world, rank, cfg.T)
    units = shard_perm(cfg.N, world, cfg.T, args.shard_mode)[n0:n0 + Nl]
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    u = torch.zeros(cfg.N, dtype=torch.int64)
    u[torch.from_numpy(units)] = 1
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(u)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "t_max": float(t.item()),
                          "units_covered_once": bool((u == 1).all()), "config": bench_config(cfg, args, world)}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def ncu_step_traffic(config: str, algo: str, launches: int, timeout: int = 300):
    """DRAM bytes of ONE forward of this build, measured now: ncu (dram__bytes_read/write.sum per kernel, caches
    not flushed between the step's kernels) on tools/prof_run.py running two forwards of the same config; the last
    `launches` kernels are the second forward.  Returns (per-kernel list, total bytes) or (None, reason)."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--csv",
           "--cache-control", "none", "--clock-control", "none", sys.executable,
           os.path.join(ROOT, "tools", "prof_run.py"), "--config", config, "--iters", "2", "--fwd", "--algo", algo]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    except subprocess.TimeoutExpired:
        return None, f"ncu timed out after {timeout} s"
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    if r.returncode != 0 or not lines:
        return None, f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-200:]}"
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}
    kern = {}
    for d in rows:
        key = (int(d["ID"]), d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        kern.setdefault(key, {})[d["Metric Name"]] = v
    ks = sorted(kern.items())[-launches:]
    out = [{"kernel": name.split("(")[0][:80], "dram_bytes": int(m.get("dram__bytes_read.sum", 0) +
                                                               m.get("dram__bytes_write.sum", 0)),
            "ncu_ms": m.get("gpu__time_duration.sum", 0.0) * 1e3} for (_, name), m in ks]
    return out, sum(k["dram_bytes"] for k in out)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="7B")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--chunks", type=int, default=4, help="M chunks overlapping compute and all-reduce (N>1)")
    ap.add_argument("--shard", choices=["hidden", "tokens"], default="hidden",
                    help="N>1: hidden-dim sharding + all-reduce (north_star (5), strong scaling) or independent "
                         "token-parallel replicas with full weights and no collective (SURVEY 8(e) control, weak scaling)")
    ap.add_argument("--allreduce", choices=["nccl", "sym", "fused"], default="nccl",
                    help="N>1: NCCL all-reduce (chunked overlap), the library's symmetric-memory reduction kernel "
                         "(NEXT-3: NVLS multimem / P2P over an NCCL symmetric window), or that reduction fused into "
                         "the DOWN GEMM per 2048-row window (union path); falls back to nccl if unsupported")
    ap.add_argument("--algo", default="auto", choices=["auto", "gather", "union"], help="fused up/down algorithm")
    ap.add_argument("--e2e-chunk", type=int, default=4096, help="rows per chunk of the host-buffer pipeline")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--shard-mode", choices=["contiguous", "round_robin"], default="contiguous",
                    help="N>1 hidden sharding: contiguous row blocks, or TwELL tiles dealt round-robin (SURVEY 8(e))")
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-run ncu pass that measures the step's DRAM bytes")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo skeleton of the multi-rank path (tests)")
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.CONFIGS[args.config]

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(sys.argv[1:], args.gpus))
    if args.dry_run:
        run_dry(args, cfg)
        return
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2603_23198_b200 as sffn

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
    from paper_2603_23198_b200.sharding import shard_perm, shard_range
    replicas = world > 1 and args.shard == "tokens"
    n0, Nl = (0, N) if replicas else shard_range(N, world, rank, T)
    units = shard_perm(N, 1 if replicas else world, T, args.shard_mode)[n0:n0 + Nl]  # this rank's hidden units

    def to_dev(a):
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev)

    p = synth.token_targets(cfg)
    X_host = synth.gen_x(cfg, p=p)
    X = to_dev(X_host)
    if args.shard_mode == "contiguous" or replicas:
        Wg, Wu, Wd = (to_dev(synth.gen_w(cfg, w, n0, Nl)) for w in "gud")
    else:  # round-robin tiles: the shard's weight rows gathered once, at load time
        Wg, Wu, Wd = (to_dev(np.ascontiguousarray(synth.gen_w(cfg, w)[units])) for w in "gud")
    Y = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    ws = torch.empty(sffn.workspace_bytes(M, K, Nl, T, C, args.algo), dtype=torch.uint8, device=dev)
    tw_view = sffn.twell_view(ws, M, Nl, C)
    ud_ws = torch.empty(max(16, sffn.up_down_workspace_bytes(M, K, Nl, T, C, args.algo)), dtype=torch.uint8, device=dev)
    ov = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    comm = sffn.Comm(rank, world, local) if world > 1 and not replicas else None
    allreduce = "none"
    if comm is not None:
        allreduce = "nccl"
        if args.allreduce in ("sym", "fused") and comm.symmetric_init(M, K):
            allreduce = ("sym-" if args.allreduce == "sym" else "fused-") + (
                "nvls" if comm.symmetric_info()["multimem"] else "p2p")

    def step():
        if comm is None:
            sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov, algo=args.algo)
        else:
            if allreduce.startswith("sym"):
                comm.sharded_forward_sym(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov, algo=args.algo)
            elif allreduce.startswith("fused"):
                comm.sharded_forward_fused(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov)
            else:
                comm.sharded_forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov, algo=args.algo,
                                     n_chunks=args.chunks)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            flush.fill_(1.0)
            fn()
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for s, e in ev:
            flush.fill_(1.0)  # L2 flush between timed steps (outside the events)
            s.record(stream)
            fn()
            e.record(stream)
        barrier()
        ms = [s.elapsed_time(e) for s, e in ev]
        return ms

    # the step is captured once into a CUDA graph (the library is capture-safe: stream-ordered, no host
    # synchronization, device-side work counts) and replayed: removes the per-launch CPU/driver gaps
    step_fn = step
    graph = None
    c0 = sffn.launch_count()
    step()  # one eager step: the library's own kernel launches per step (host-side counter of the .so)
    launches_per_step = sffn.launch_count() - c0
    torch.cuda.synchronize()
    if not args.no_graph and world == 1:
        for _ in range(2):
            step()  # first calls set kernel attributes outside the capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        step_fn = graph.replay

    # ------------------------------------------------------------------ main timed region
    clocks = Clocks(local)
    clocks.start()
    ms = timed(step_fn, args.steps, args.warmup)
    clk = clocks.stop()
    # warm-L2 steps (no flush between them), reported separately; not the headline value
    barrier()
    ev_w = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(max(3, args.steps // 4))]
    for s_, e_ in ev_w:
        s_.record(stream)
        step_fn()
        e_.record(stream)
    barrier()
    warm_ms = float(np.median([s_.elapsed_time(e_) for s_, e_ in ev_w]))
    n_ov = sffn.overflow_check(ov)
    t_local = float(np.sum(ms)) / 1e3
    t_max = t_local
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_per_step = t_max / args.steps * 1e3
    # tokens/s, whole job: hidden-dim sharding -> all ranks jointly process the M tokens; replicas -> M each
    value = (world if replicas else 1) * M * args.steps / t_max

    # ------------------------------------------------------------------ per-kernel timing (roofline)
    peaks = load_peaks()
    tw = torch.empty((M, Nl // C), dtype=torch.int32, device=dev)
    ms_pack = timed(lambda: sffn.pack(X, Wg, T, C, out=tw), max(5, args.steps // 2), 3)
    ms_ud = timed(lambda: sffn.up_down(X, tw, Wu, Wd, T, C, out=Y, workspace=ud_ws, algo=args.algo),
                  max(5, args.steps // 2), 3)
    c0 = sffn.launch_count()
    sffn.up_down(X, tw, Wu, Wd, T, C, out=Y, workspace=ud_ws, algo=args.algo)
    ud_launches = sffn.launch_count() - c0
    t_pack = float(np.median(ms_pack)) / 1e3
    t_ud = float(np.median(ms_ud)) / 1e3
    twords = tw.cpu().numpy().view(np.uint32).reshape(M, Nl // T, T // C)
    tile_cnt = np.minimum(twords[:, :, 0], T // C - 1).astype(np.int64)
    nnz_row = tile_cnt.sum(1)
    nnz_total = int(nnz_row.sum())
    # realized activation statistics of this run (SURVEY §8d-3 outputs): per-token nnz quantiles and the per-tile
    # count histogram (counts 0..cap, plus overflowed tiles)
    hist = np.bincount(np.minimum(twords[:, :, 0], T // C).astype(np.int64).ravel(), minlength=T // C + 1)
    nnz_stats = {"mean": float(nnz_row.mean()), "p50": float(np.median(nnz_row)),
                 "p99": float(np.percentile(nnz_row, 99)), "max": int(nnz_row.max()),
                 "realized_sparsity": 1.0 - nnz_total / (M * Nl),
                 "tile_count_hist": {"bins": f"count 0..{T // C - 1}, then >= {T // C} (overflow)",
                                     "counts": [int(v) for v in hist]}}
    gate_flop = 2.0 * M * K * Nl
    ud_flop = 4.0 * K * nnz_total  # useful sparse work of Eq.3
    ud_compulsory = 2 * M * K + 4 * M * Nl // C + 2 * M * K + 4 * Nl * K  # x, TwELL, y, touched weights (<=)
    fma_peak = N_SMS * FMA_LANES_PER_SM * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    kernels = {
        "gate_gemm_twell": {"ms": t_pack * 1e3, "launches": 1, "bound": "tensor",
                            "achieved": gate_flop / t_pack / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                            "frac": gate_flop / t_pack / 1e12 / peaks["bf16_tflops"],
                            "algorithmic": "2*M*K*N FLOP"},
    }
    algo_used = args.algo if args.algo != "auto" else ("union" if Nl % 64 == 0 else "gather")
    # SURVEY §8d-4 floor of the fused up/down (K2'): the method's useful work 4 K nnz FLOP at the FP32-FMA peak vs
    # its compulsory bytes at the HBM copy bandwidth; frac = floor / measured
    t_floor_ud = max(ud_flop / (fma_peak * 1e12), ud_compulsory / (peaks["hbm_gbs"] * 1e9))
    if algo_used == "union":
        st = sffn.union_stats(ud_ws, M, K, Nl)
        br = st["block_rows"]
        tc_flop = 4.0 * br * st["padded_sum"] * K  # the two union GEMMs
        kernels["fused_up_down"] = {
            "ms": t_ud * 1e3, "launches": ud_launches, "algo": "union", "bound": "alu",
            "achieved": ud_flop / t_ud / 1e12, "peak": fma_peak, "unit": "TFLOP/s",
            "frac": t_floor_ud / t_ud, "floor_ms": t_floor_ud * 1e3,
            "algorithmic": "4*K*nnz FLOP (Eq.3 useful work), floor = max(FLOP / FP32-FMA peak, compulsory bytes / HBM)",
            "tensor_padded": {"achieved": tc_flop / t_ud / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                              "frac": tc_flop / t_ud / 1e12 / peaks["bf16_tflops"],
                              "work": f"4*{br}*sum_b |U_b| * K FLOP executed by the union GEMMs ({br}-row blocks)",
                              "redundancy": tc_flop / max(ud_flop, 1.0)},
            "union_frac_of_N": st["union_sum"] / ((M + br - 1) // br) / Nl, "union_block_rows": br}
        # the union GEMMs' operand stream (the resource that bounds them): UP reads an A tile (X rows, 128 x 64 bf16)
        # per k-block of each (block, chunk) tile and every union row of W_u once per block; DOWN an A tile (H_c) per
        # k-block of each (block, column tile) and every union row of W_d once per block
        kb_bytes = 128 * 64 * 2
        ingress = (st["up_tiles"] * (K // 64) * kb_bytes + st["padded_sum"] * K * 2
                   + ((K + 255) // 256) * (st["padded_sum"] // 64) * kb_bytes + st["padded_sum"] * K * 2)
        clk_mhz = (clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0))
        t_ud_gemm = t_ud  # includes the prep kernel: a conservative (lower) fraction
        kernels["fused_up_down"]["ingress"] = {
            "bound": "l2_to_sm_ingress", "bytes": ingress, "unit": "B/cycle/SM",
            "achieved": ingress / t_ud_gemm / (N_SMS * clk_mhz * 1e6), "peak": INGRESS_B_PER_CYCLE_SM,
            "frac": ingress / t_ud_gemm / (N_SMS * clk_mhz * 1e6) / INGRESS_B_PER_CYCLE_SM,
            "clock_mhz": clk_mhz,
            "what": "A tiles + gathered weight rows of both union GEMMs per step over the whole up/down time (prep "
                    "included) at the bench's median SM clock, vs the measured per-SM ingress ceiling"}
    else:
        kernels["fused_up_down"] = {
            "ms": t_ud * 1e3, "launches": ud_launches, "algo": "gather", "bound": "alu", "achieved": ud_flop / t_ud / 1e12,
            "peak": fma_peak, "unit": "TFLOP/s", "frac": t_floor_ud / t_ud, "floor_ms": t_floor_ud * 1e3,
            "algorithmic": "4*K*nnz FLOP", "hbm_compulsory_gbs": ud_compulsory / t_ud / 1e9,
            "gathered_gbs": 4.0 * K * nnz_total / t_ud / 1e9}
    # the dominant single launch: the gate GEMM (the union up/down is several launches, none longer than it;
    # see profiles/ launch lists); the gather kernel is one launch and longer than the gate GEMM
    dom = "gate_gemm_twell" if (algo_used == "union" or t_pack >= t_ud) else "fused_up_down"
    traffic = None
    hbm = None
    step_kernels = None
    if rank == 0 and world == 1 and not args.no_ncu:
        # the metric's "HBM %": DRAM bytes of one forward of THIS build, measured now by an ncu pass (only DRAM byte
        # counters are taken from it, never a time), over the step time measured above
        step_kernels, tot = ncu_step_traffic(args.config, args.algo, launches_per_step)
        if step_kernels is None:
            hbm = {"unavailable": tot}
        else:
            hbm = {"step_dram_bytes": tot, "achieved_gbs": tot / (ms_per_step / 1e3) / 1e9, "peak_gbs": peaks["hbm_gbs"],
                   "frac": tot / (ms_per_step / 1e3) / 1e9 / peaks["hbm_gbs"],
                   "frac_spec_8tbs": tot / (ms_per_step / 1e3) / 1e9 / 8000.0,
                   "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one forward, measured in this run "
                             "(--cache-control none), / the bench step time", "kernels": step_kernels}
            gate = [k for k in step_kernels if "gemm_tc_kernel" in k["kernel"]]
            if dom == "gate_gemm_twell" and gate:
                traffic = gate[0]["dram_bytes"]
    kd = kernels[dom]
    roofline = {"bound": kd["bound"], "achieved": kd["achieved"], "peak": kd["peak"], "unit": kd["unit"],
                "frac": kd["frac"], "traffic": traffic, "kernel": dom,
                "peak_source": peaks["_source"] + " burst" if kd["bound"] == "tensor" else
                "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz (DESIGN.md)"}
    if kd["bound"] == "tensor":
        # the measured cuBLAS burst figure is below what this kernel reaches (frac > 1); the nominal dense bf16 peak
        # (B200_PROFILING.md: 2.25 PFLOP/s at boost clock) and the algorithmic bytes are given for interpretation
        roofline["nominal_peak"] = 2250.0
        roofline["frac_nominal"] = kd["achieved"] / 2250.0
        roofline["algorithmic_bytes"] = float(2 * M * K + 2 * Nl * K + 4 * M * Nl // C)  # X + W_g + TwELL

    # ------------------------------------------------------------------ dense baseline (own tcgen05 FFN)
    dense = None
    if not args.no_dense and world == 1:
        wdT = sffn.transpose(Wd)
        H = torch.empty((M, Nl), dtype=torch.bfloat16, device=dev)
        Yd = torch.empty_like(Y)
        ms_d = timed(lambda: sffn.dense_forward(X, Wg, Wu, wdT, h=H, out=Yd), max(5, args.steps // 2), 3)
        t_d = float(np.median(ms_d)) / 1e3
        dense = {"ms_per_step": t_d * 1e3, "tokens_per_s": M / t_d, "tflops": 6.0 * M * K * Nl / t_d / 1e12,
                 "speedup_sparse_vs_dense": t_d / (ms_per_step / 1e3)}
        # sanity line for the denominator's quality: the same three GEMMs through torch.matmul
        # (cuBLAS), H taken as given (no GLU epilogue)
        G1 = torch.empty((M, Nl), dtype=torch.bfloat16, device=dev)
        ms_t = timed(lambda: (torch.matmul(X, Wg.t(), out=G1), torch.matmul(X, Wu.t(), out=H),
                              torch.matmul(H, Wd, out=Yd)), max(5, args.steps // 2), 3)
        t_t = float(np.median(ms_t)) / 1e3
        dense["torch_matmul"] = {"ms_per_step": t_t * 1e3, "tflops": 6.0 * M * K * Nl / t_t / 1e12,
                                 "what": "torch.matmul (cuBLAS) X W_g^T, X W_u^T, H W_d: the dense FFN's three GEMMs "
                                         "without the GLU epilogue"}
        del H, Yd, wdT, G1

    # ------------------------------------------------------------------ end to end (host buffers)
    e2e = None
    if not args.no_e2e and world == 1:
        # through the public host-buffer API: pinned X in, pinned Y out, copies inside the timed region
        Xh = torch.from_numpy(X_host.view(np.int16)).view(torch.bfloat16).pin_memory()
        Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
        rows = min(args.e2e_chunk, M)
        wsz = sffn.workspace_bytes(rows, K, Nl, T, C, args.algo)  # two: chunks alternate two compute streams
        ws_h = torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device=dev)
        stage = torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, ((rows + 127) // 128) * 128)),
                            dtype=torch.uint8, device=dev)

        def e2e_step():
            sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=ws_h, stage=stage, overflow=ov,
                              algo=args.algo, chunk_rows=args.e2e_chunk, synchronize=False)

        ms_e = timed(e2e_step, max(3, args.steps // 3), 3)
        t_e = float(np.sum(ms_e)) / 1e3
        e2e = {"value": M * len(ms_e) / t_e, "unit": "tokens/s", "h2d_bytes_per_step": int(Xh.numel() * 2),
               "d2h_bytes_per_step": int(Yh.numel() * 2), "ms_per_step": t_e / len(ms_e) * 1e3,
               "api": f"sffn_forward_host (pinned host X/Y, chunks of {args.e2e_chunk} rows, copy/compute overlap)"}
        del ws_h, stage
    elif not args.no_e2e and world > 1:
        # N > 1: every rank copies X from pinned host memory, runs the sharded forward through the public API
        # (Comm.sharded_forward / sharded_forward_sym), and copies Y back; copies inside the timed region (serial,
        # no overlap); max over ranks as for `value`
        Xh = torch.from_numpy(X_host.view(np.int16)).view(torch.bfloat16).pin_memory()
        Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
        Xd = torch.empty_like(X)

        def e2e_step():
            Xd.copy_(Xh, non_blocking=True)
            if replicas:
                sffn.forward(Xd, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov, algo=args.algo)
            elif allreduce.startswith("sym"):
                comm.sharded_forward_sym(Xd, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov, algo=args.algo)
            elif allreduce.startswith("fused"):
                comm.sharded_forward_fused(Xd, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov)
            else:
                comm.sharded_forward(Xd, Wg, Wu, Wd, T, C, out=Y, workspace=ws, overflow=ov, algo=args.algo,
                                     n_chunks=args.chunks)
            Yh.copy_(Y, non_blocking=True)

        ms_e = timed(e2e_step, max(3, args.steps // 3), 3)
        t_e = float(np.sum(ms_e)) / 1e3
        tt = torch.tensor([t_e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e = float(tt.item())
        e2e = {"value": (world if replicas else 1) * M * len(ms_e) / t_e, "unit": "tokens/s",
               "h2d_bytes_per_step": int(Xh.numel() * 2),
               "d2h_bytes_per_step": int(Yh.numel() * 2), "ms_per_step": t_e / len(ms_e) * 1e3,
               "api": ("sffn.forward" if replicas else "Comm.sharded_forward") + " on every rank with X copied in from pinned host memory and Y copied out "
                      "(serial copies; per-rank bytes)"}

    # ------------------------------------------------------------------ CPU oracle baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(cfg, p, target_s=12.0)

    if comm is not None:
        comm.close()
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong" if world > 1 and not replicas else "weak", "vs_baseline": None, "dtype": "bf16",
               "data": DATA,
               "config": bench_config(cfg, args, world),
               "tokens_per_s_per_gpu": value / world, "allreduce_used": allreduce,
               "launch_used": "cuda_graph" if graph is not None else "eager",
               "roofline": roofline, "kernels": kernels, "nnz_per_token": nnz_total / M, "nnz": nnz_stats,
               "overflow_tiles": n_ov, "dense": dense, "e2e": e2e, "cpu_baseline": cpu,
               "hbm": hbm,
               "warm_l2_ms_per_step": warm_ms,
               "gpu_launches": args.steps * launches_per_step,
               "gpu_launches_per_step": launches_per_step,
               "algo": algo_used,
               "clocks": clk}
        line = json.dumps(out)
        print(line, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(line + "\n")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
