"""Child process of test_sharded_forward_fused_single_rank (run under a timeout: a counter that never reaches its
target would spin forever).  Fused window-granular all-reduce on a 1-rank communicator vs sffn_forward (union);
prints OK."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__))]
import torch  # noqa: E402

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import assert_y, to_dev  # noqa: E402


def main():
    import paper_2603_23198_b200 as sffn
    comm = sffn.Comm(0, 1, torch.cuda.current_device())
    try:
        # M > 2 windows with a ragged last window and a ragged last 128-row block; K = 640: a ragged column tile
        cfg = synth.CONFIGS["1B"].replace(M=4500, K=640, N=2048, Kb=32, sparsity=0.97)
        if not comm.symmetric_init(8192, cfg.K):
            print("SKIP symmetric windows unsupported")
            return
        Xn, Wgn, Wun, Wdn = synth.gen_x(cfg), synth.gen_w(cfg, "g"), synth.gen_w(cfg, "u"), synth.gen_w(cfg, "d")
        X, Wg, Wu, Wd = (to_dev(a) for a in (Xn, Wgn, Wun, Wdn))
        ref = sffn.forward(X, Wg, Wu, Wd, 256, 8, algo="union")
        words, counts, n_ov, A = oracle.pack_from_inputs(Xn, Wgn, 256, 8)
        Y3 = oracle.ffn_twell(Xn, words, Wun, Wdn, cfg.N, 256, 8)
        print("ref done", flush=True)
        for it in range(3):  # the counters are never reset: each call raises the targets by one epoch
            Y = comm.sharded_forward_fused(X, Wg, Wu, Wd, 256, 8)
            torch.cuda.synchronize()
            print("call", it, "max diff", (Y.float() - ref.float()).abs().max().item(), flush=True)
            assert torch.equal(Y.view(torch.int16), ref.view(torch.int16)), f"call {it}"
            assert_y(Y.float().cpu().numpy().astype(np.float64), Y3)  # the oracle of the (1-rank) problem
        # a smaller M on the same window (one partial window), then the large one again
        for rows in (1000, 4500, 1):
            ref_r = sffn.forward(X[:rows].contiguous(), Wg, Wu, Wd, 256, 8, algo="union")
            Y = comm.sharded_forward_fused(X[:rows].contiguous(), Wg, Wu, Wd, 256, 8)
            torch.cuda.synchronize()
            assert torch.equal(Y.view(torch.int16), ref_r.view(torch.int16)), f"rows {rows}"
        # captured into a CUDA graph and replayed: the counter set alternates on the device
        Yg = torch.empty_like(ref)
        wsg = torch.empty(sffn.workspace_bytes(cfg.M, cfg.K, cfg.N, 256, 8, "union"), dtype=torch.uint8, device="cuda")
        comm.sharded_forward_fused(X, Wg, Wu, Wd, 256, 8, out=Yg, workspace=wsg)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            comm.sharded_forward_fused(X, Wg, Wu, Wd, 256, 8, out=Yg, workspace=wsg)
        for it in range(3):
            Yg.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(Yg.view(torch.int16), ref.view(torch.int16)), f"replay {it}"
        print("graph replays ok", flush=True)
        try:
            comm.sharded_forward_fused(torch.zeros(9000, cfg.K, dtype=torch.bfloat16, device="cuda"), Wg, Wu, Wd)
            raise AssertionError("M above the window accepted")
        except sffn.SffnError:
            pass
        print("OK")
    finally:
        comm.close()


if __name__ == "__main__":
    main()
