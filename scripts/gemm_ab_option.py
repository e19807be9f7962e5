"""A/B one GEMM option on the same box, interleaved rounds (power-cap drift
hits both arms alike), with cuBLAS beside them; the two arms' outputs must
be bit-identical and match cuBLAS.

    python scripts/gemm_ab_option.py gemm_dynamic 0 1 [M,N,K ...]

profiles/r2_gemm_early_ab.log is a negative result kept for the record: an
experimental wide-kernel option that started the next tile's half-0 UMMAs
while the epilogue drained half 1 was bit-identical but not faster
(-3% .. +1%, within the power-cap noise), so it was not kept.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402


def t(fn, reps=10):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


name, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[4:]] or [
    (8192, 8192, 8192), (16384, 65536, 8192), (16384, 32768, 8192), (16384, 8192, 65536),
    (10240, 16384, 4096), (10240, 4096, 16384)]
st = torch.cuda.current_stream().cuda_stream
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
    outs = {v: torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for v in (va, vb)}
    ref = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    def ours(v):
        with C.option(name, v):
            C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), outs[v].data_ptr(),
                                           M, N, K, 0, st), "gemm")

    res = {va: [], vb: [], "cublas": []}
    for _ in range(4):
        res[va].append(t(lambda: ours(va)))
        res[vb].append(t(lambda: ours(vb)))
        res["cublas"].append(t(lambda: torch.matmul(a, b, out=ref)))
    assert torch.equal(outs[va], outs[vb]), (M, N, K)
    err = ((outs[vb].float() - ref.float()).abs().max() / ref.float().abs().max()).item()
    assert err < 8e-3, err
    f = 2.0 * M * N * K
    print(json.dumps({"M": M, "N": N, "K": K, "option": name, "bit_identical": True,
                      "rel_vs_cublas": err,
                      f"tflops_{name}={va}": round(f / min(res[va]) / 1e9, 1),
                      f"tflops_{name}={vb}": round(f / min(res[vb]) / 1e9, 1),
                      "tflops_cublas": round(f / min(res["cublas"]) / 1e9, 1)}), flush=True)
    del a, b, outs, ref
    torch.cuda.empty_cache()
