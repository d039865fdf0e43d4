"""Child process of test_fused_allreduce_emulated: G "ranks" of the fused all-reduce on ONE GPU, without NCCL.
Each rank gets its own window (plain device buffer: partial Y + two counter sets) and its own hidden shard; the
pointer table lists the G windows, no multicast.  Phase 1 (pack, metadata, UP) runs rank by rank; then the G fused
DOWN kernels run concurrently on G streams, each on 1/G of the SMs (SFFN_UNION_GRID), so the window counters, the
owner mapping (w mod G) and the P2P reduction across G windows run as on G GPUs.  Expected: every window holds
bf16(sum_r fp32(P_r)) with P_r = sffn_forward of rank r's shard, the reducer's summation order, AND the reduced Y is
within the Y bar (per row 1e-2) of the oracle's Eq.3 / Eq.1 of the UNSHARDED problem.  The forward runs twice: the
second call uses the other counter set (the table's set offset flipped and the first set zeroed on the host, as the
finish kernel does on the device).  argv: G [contiguous|round_robin].  Prints OK."""
import os
import sys

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
MODE = sys.argv[2] if len(sys.argv) > 2 else "contiguous"
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__))]
import torch  # noqa: E402

os.environ["SFFN_UNION_GRID"] = str(torch.cuda.get_device_properties(0).multi_processor_count // G)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import ROW_TOL_EQ1, assert_y, to_dev  # noqa: E402


def main():
    import paper_2603_23198_b200 as sffn
    from paper_2603_23198_b200.sffn import lib
    from paper_2603_23198_b200.sharding import shard_perm
    L = lib()
    f = L.sffn__forward_fused  # signature bound by the package (internal entry, include/sffn.h)
    Nl = 1024
    cfg = synth.CONFIGS["1B"].replace(M=4500, K=640, N=Nl * G, Kb=32, sparsity=0.97)
    M, K, T, C = cfg.M, cfg.K, 256, 8
    Xn, Wgn, Wun, Wdn = synth.gen_x(cfg), synth.gen_w(cfg, "g"), synth.gen_w(cfg, "u"), synth.gen_w(cfg, "d")
    X = to_dev(Xn)
    Wg, Wu, Wd = to_dev(Wgn), to_dev(Wun), to_dev(Wdn)
    perm = torch.from_numpy(shard_perm(cfg.N, G, T, MODE)).cuda()
    sh = [tuple(W[perm[r * Nl:(r + 1) * Nl]].contiguous() for W in (Wg, Wu, Wd)) for r in range(G)]
    flags_off = (M * K * 2 + 255) // 256 * 256
    nwin = (M + 2047) // 2048
    wins = [torch.zeros(flags_off + 8 * nwin, dtype=torch.uint8, device="cuda") for _ in range(G)]
    table = torch.tensor([w.data_ptr() for w in wins] + [0, flags_off], dtype=torch.int64, device="cuda")
    wsz = sffn.workspace_bytes(M, K, Nl, T, C, "union")
    ws = [torch.empty(wsz, dtype=torch.uint8, device="cuda") for _ in range(G)]
    cur = torch.cuda.current_stream()

    def call(r, phase, stream):
        st = f(X.data_ptr(), sh[r][0].data_ptr(), sh[r][1].data_ptr(), sh[r][2].data_ptr(), M, K, Nl, T, C,
               wins[r].data_ptr(), ws[r].data_ptr(), wsz, None, table.data_ptr(), G, r, phase, stream.cuda_stream)
        assert st == 0, f"sffn__forward_fused rank {r} phase {phase}: status {st}"

    acc = None
    for r in range(G):
        P = sffn.forward(X, *sh[r], T, C, algo="union").float()
        acc = P if acc is None else acc + P
    ref = acc.to(torch.bfloat16)
    words, counts, n_ov, A = oracle.pack_from_inputs(Xn, Wgn, T, C)
    Y3 = oracle.ffn_twell(Xn, words, Wun, Wdn, cfg.N, T, C)  # Eq.3 of the unsharded problem
    ok = ~(counts > T // C - 1).any(1)                         # rows without an overflowed tile (reading R5)
    assert ok.sum() > M // 2
    Y1 = oracle.ffn_dense(Xn[ok], Wgn, Wun, Wdn)              # Eq.1 on those rows
    streams = [torch.cuda.Stream() for _ in range(G)]
    for call_i, cset in enumerate((0, 1)):
        off = flags_off + 4 * nwin * cset
        for w in wins:
            w[:flags_off].zero_()
        for r in range(G):
            call(r, 1, cur)
        torch.cuda.synchronize()
        for r in range(G):
            call(r, 2, streams[r])
        torch.cuda.synchronize()
        print(f"call {call_i}: fused DOWN kernels done (counter set {cset})", flush=True)
        for r in range(G):
            Y = wins[r][:M * K * 2].view(torch.bfloat16).view(M, K)
            bad = (Y.view(torch.int16) != ref.view(torch.int16)).sum().item()
            assert bad == 0, f"window {r}: {bad} elements differ from bf16(sum of partials)"
            cnt = wins[r][off:off + 4 * nwin].view(torch.int32).cpu().tolist()
            want = [4 * ((min(2048, M - w * 2048) + 127) // 128) * ((K + 255) // 256) * G if w % G == r else 0
                    for w in range(nwin)]
            assert cnt == want, f"window {r} set {cset} counters {cnt} != {want}"
            y = Y.float().cpu().numpy().astype(np.float64)
            assert_y(y, Y3)
            assert_y(y[ok], Y1, row_tol=ROW_TOL_EQ1)
        # what sym_finish_kernel does after its barrier: zero the set this call used, flip the table's set offset
        for w in wins:
            w[off:off + 4 * nwin].zero_()
        table[G + 1] = flags_off + 4 * nwin * (1 - cset)
        torch.cuda.synchronize()
    print("OK", flush=True)


if __name__ == "__main__":
    main()
