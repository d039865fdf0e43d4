"""Child process of test_fused_allreduce_emulated: G "ranks" of the fused all-reduce on ONE GPU, without NCCL.
Each rank gets its own window (plain device buffer: partial Y + two counter sets) and its own hidden shard; the
pointer table lists the G windows, no multicast.  Phase 1 (pack, metadata, UP) runs rank by rank; then the G fused
DOWN kernels run concurrently on G streams, each on 1/G of the SMs (SFFN_UNION_GRID), so the window counters, the
owner mapping (w mod G) and the P2P reduction across G windows run as on G GPUs.  Expected: every window holds
bf16(sum_r fp32(P_r)) with P_r = sffn_forward of rank r's shard, the reducer's summation order.  Prints OK."""
import os
import sys

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__))]
import torch  # noqa: E402

os.environ["SFFN_UNION_GRID"] = str(torch.cuda.get_device_properties(0).multi_processor_count // G)
import synth  # noqa: E402
from gpu_util import to_dev  # noqa: E402


def main():
    import paper_2603_23198_b200 as sffn
    from paper_2603_23198_b200.sffn import lib
    L = lib()
    f = L.sffn__forward_fused  # signature bound by the package (internal entry, include/sffn.h)
    Nl = 1024
    cfg = synth.CONFIGS["1B"].replace(M=4500, K=640, N=Nl * G, Kb=32, sparsity=0.97)
    M, K, T, C = cfg.M, cfg.K, 256, 8
    X = to_dev(synth.gen_x(cfg))
    Wg, Wu, Wd = (to_dev(synth.gen_w(cfg, w)) for w in "gud")
    sh = [(Wg[r * Nl:(r + 1) * Nl].contiguous(), Wu[r * Nl:(r + 1) * Nl].contiguous(),
           Wd[r * Nl:(r + 1) * Nl].contiguous()) for r in range(G)]
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

    for r in range(G):
        call(r, 1, cur)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(G)]
    for r in range(G):
        call(r, 2, streams[r])
    torch.cuda.synchronize()
    print("fused DOWN kernels done", flush=True)
    acc = None
    for r in range(G):
        P = sffn.forward(X, *sh[r], T, C, algo="union").float()
        acc = P if acc is None else acc + P
    ref = acc.to(torch.bfloat16)
    for r in range(G):
        Y = wins[r][:M * K * 2].view(torch.bfloat16).view(M, K)
        bad = (Y.view(torch.int16) != ref.view(torch.int16)).sum().item()
        assert bad == 0, f"window {r}: {bad} elements differ from bf16(sum of partials)"
        cnt = wins[r][flags_off:flags_off + 4 * nwin].view(torch.int32).cpu().tolist()
        want = [4 * ((min(2048, M - w * 2048) + 127) // 128) * ((K + 255) // 256) * G if w % G == r else 0
                for w in range(nwin)]
        assert cnt == want, f"window {r} counters {cnt} != {want}"
    print("OK", flush=True)


if __name__ == "__main__":
    main()
