#!/usr/bin/env python
"""Benchmark of the sparse gated-FFN forward (TwELL) on B200 — prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7B] [--impl ours|reference]

A step = one pass of the whole hot path (pack: gate GEMM -> TwELL, then the fused sparse up/down; plus
the NCCL all-reduce of partial outputs when N > 1) over one batch of M synthetic tokens, inputs and
weights resident in HBM.  The L2 is flushed (a 512 MiB write) between timed steps; every step is timed
with CUDA events on the launching stream; the reported time is the max over ranks.

N > 1 (torchrun): hidden-dim sharding (north_star (5)) — rank r owns hidden units [r N/G, (r+1) N/G) of
all three weights; every rank sees all M tokens; value = M / t (strong scaling: total work fixed).

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
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
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
def time_oracle(cfg, rows: int, p=None):
    """The oracle as it stands (pack_from_inputs + ffn_twell) on `rows` contiguous token rows."""
    import oracle
    X = synth.gen_x(cfg, 0, rows, p=p)
    Wg, Wu, Wd = synth.gen_w(cfg, "g"), synth.gen_w(cfg, "u"), synth.gen_w(cfg, "d")
    t0 = time.perf_counter()
    words, counts, ov, A = oracle.pack_from_inputs(X, Wg, cfg.T, cfg.C)
    oracle.ffn_twell(X, words, Wu, Wd, cfg.N, cfg.T, cfg.C)
    return time.perf_counter() - t0


def oracle_sample_rows(cfg, target_s: float = 15.0):
    """Rows of CPU work of about target_s seconds: calibrate on a few rows, then scale (rows are independent)."""
    ncpu = os.cpu_count() or 1
    r0 = max(1, min(ncpu, 8))
    t = time_oracle(cfg, r0)
    rows = int(max(r0, min(cfg.M, r0 * target_s / max(t, 1e-3))))
    rows = max(r0, (rows // ncpu) * ncpu) if rows >= ncpu else rows
    return rows, t, r0


def run_reference(args, cfg):
    """--impl reference: the CPU oracle, each step a bounded row sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncpu = os.cpu_count() or 1
    p = synth.token_targets(cfg)
    # one step ~ a few seconds of oracle work so the whole run stays within minutes
    rows, t_cal, r_cal = oracle_sample_rows(cfg, target_s=max(1.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        time_oracle(cfg, rows, p)
    times = [time_oracle(cfg, rows, p) for _ in range(args.steps)]
    t = float(np.mean(times))
    val = rows / t
    sample = f"{rows} contiguous token rows of {cfg.name} (M={cfg.M}) per step; fp64 gate GEMM + Alg.1 pack + Eq.3"
    out = {"metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "none",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded dyadic-grid generator)",
           "config": {"workload": cfg.name, "M": cfg.M, "K": cfg.K, "N": cfg.N, "T": cfg.T, "C": cfg.C,
                      "sparsity": cfg.sparsity},
           "impl": "reference",
           "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": min(ncpu, rows), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


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
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.CONFIGS[args.config]

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
    from paper_2603_23198_b200.sharding import shard_range
    replicas = world > 1 and args.shard == "tokens"
    n0, Nl = (0, N) if replicas else shard_range(N, world, rank, T)

    def to_dev(a):
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev)

    p = synth.token_targets(cfg)
    X_host = synth.gen_x(cfg, p=p)
    X = to_dev(X_host)
    Wg, Wu, Wd = (to_dev(synth.gen_w(cfg, w, n0, Nl)) for w in "gud")
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
    nnz_total = int(np.minimum(twords[:, :, 0], T // C - 1).sum())
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
    if algo_used == "union":
        st = sffn.union_stats(ud_ws, M, K, Nl)
        br = st["block_rows"]
        tc_flop = 4.0 * br * st["padded_sum"] * K  # the two union GEMMs
        kernels["fused_up_down"] = {
            "ms": t_ud * 1e3, "launches": ud_launches, "algo": "union", "bound": "tensor",
            "achieved": tc_flop / t_ud / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
            "frac": tc_flop / t_ud / 1e12 / peaks["bf16_tflops"],
            "algorithmic": f"4*{br}*sum_b |U_b| * K FLOP (union GEMMs, {br}-row union blocks)",
            "union_frac_of_N": st["union_sum"] / ((M + br - 1) // br) / Nl, "union_block_rows": br,
            "useful_tflops": ud_flop / t_ud / 1e12}
    else:
        kernels["fused_up_down"] = {
            "ms": t_ud * 1e3, "launches": ud_launches, "algo": "gather", "bound": "alu", "achieved": ud_flop / t_ud / 1e12,
            "peak": fma_peak, "unit": "TFLOP/s", "frac": ud_flop / t_ud / 1e12 / fma_peak,
            "algorithmic": "4*K*nnz FLOP", "hbm_compulsory_gbs": ud_compulsory / t_ud / 1e9,
            "gathered_gbs": 4.0 * K * nnz_total / t_ud / 1e9}
    # the dominant single launch: the gate GEMM (the union up/down is several launches, none longer than it;
    # see profiles/ launch lists); the gather kernel is one launch and longer than the gate GEMM
    dom = "gate_gemm_twell" if (algo_used == "union" or t_pack >= t_ud) else "fused_up_down"
    traffic = None
    hbm = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tr = json.load(f)
            traffic = tr.get(args.config, {}).get(dom)
            # the metric's "HBM %": DRAM bytes of the step's kernels (one ncu --set full capture of the same
            # forward, tools/prof_step.sh) over the measured step time, against the measured copy bandwidth
            step_k = (["gate_gemm_twell", "union_rank", "permute_rows", "union_meta", "union_gate_list",
                       "union_up_gemm", "union_down_gemm"] if algo_used == "union" else [])
            tk = tr.get(args.config, {})
            if world == 1 and step_k and all(k in tk for k in step_k):
                b = float(sum(tk[k] for k in step_k))
                hbm = {"step_dram_bytes": b, "achieved_gbs": b / (ms_per_step / 1e3) / 1e9,
                       "peak_gbs": peaks["hbm_gbs"], "frac": b / (ms_per_step / 1e3) / 1e9 / peaks["hbm_gbs"],
                       "source": "ncu dram__bytes_read+write per kernel (profiles/ncu_traffic.json) / bench step time"}
        except (OSError, ValueError):
            traffic = None
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
        del H, Yd, wdT

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
                              algo=args.algo, chunk_rows=args.e2e_chunk)

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
        rows, _, _ = oracle_sample_rows(cfg, target_s=12.0)
        t_o = time_oracle(cfg, rows, p)
        cpu = {"value": rows / t_o, "unit": "tokens/s", "cores": min(os.cpu_count() or 1, rows), "kind": "oracle",
               "sample": f"{rows} contiguous token rows of {cfg.name}: fp64 gate GEMM + Alg.1 pack + Eq.3 "
                         f"({t_o:.1f} s)"}

    if comm is not None:
        comm.close()
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong" if world > 1 and not replicas else "weak", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic (seeded dyadic-grid generator: 99% sparsity, lognormal per-token nnz, "
                       "30% dead neurons)",
               "config": {"workload": cfg.name, "M": M, "K": K, "N": N, "T": T, "C": C, "sparsity": cfg.sparsity,
                          "parallelism": (f"token replicas x{world}" if replicas else f"hidden-dim x{world}")
                          if world > 1 else "single", "allreduce": allreduce,
                          "l2": "flushed (512 MiB write) between timed steps", "seed": cfg.seed,
                          "launch": "cuda_graph" if graph is not None else "eager"},
               "tokens_per_s_per_gpu": value / world,
               "roofline": roofline, "kernels": kernels, "nnz_per_token": nnz_total / M,
               "overflow_tiles": n_ov, "dense": dense, "e2e": e2e, "cpu_baseline": cpu,
               "hbm": hbm,
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
