"""GEMM slowdown under a concurrent gather (2 ranks): our tcgen05 GEMM alone vs
with a concurrent (a) local copy-engine copy, (b) peer all-gather on the copy
engines, (c) peer all-gather with the background SM pull (32 CTAs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2105_04663_b200 import _capi as C
from paper_2105_04663_b200.executor import NcclComm, _groups_arg, desc
from paper_2105_04663_b200.ir import DType, Shape
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
comm = NcclComm.from_torch_distributed()
lib = C.lib()
comm.ensure_peer(600 << 20, dev)
M, N, K = 8192, 32768, 8192
a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
b = torch.randn(K, N, device=dev, dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
main = torch.cuda.current_stream(); side = torch.cuda.Stream(device=dev)
src = torch.randn(128 << 20, device=dev, dtype=torch.bfloat16)   # 256 MB
dst = torch.empty(world * (128 << 20), device=dev, dtype=torch.bfloat16)
garr, ng, gs = _groups_arg([list(range(world))])
sh_in, sh_out = Shape((128 << 20,), DType.BF16), Shape((world * (128 << 20),), DType.BF16)
def gemm():
    C.check(lib.spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, main.cuda_stream), "g")
def bg(kind):
    with torch.cuda.stream(side):
        if kind == "local_ce":
            dst[: 128 << 20].copy_(src, non_blocking=True)
        elif kind in ("peer_ce", "peer_sm"):
            C.check(lib.spmd_peer_all_gather(comm.handle, desc(src.view(1, -1), sh_in), desc(dst.view(1, -1), sh_out),
                                             0, garr, ng, gs, 0, 1, 0 if kind == "peer_ce" else 3, side.cuda_stream), "ag")
res = {}
for kind in ["none", "local_ce", "peer_ce", "peer_sm", "none"]:
    times = []
    for it in range(6):
        torch.cuda.synchronize(); dist.barrier()
        side.wait_stream(main)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        if kind != "none": bg(kind)
        gemm()
        e1.record(main)
        main.wait_stream(side)
        torch.cuda.synchronize()
        if it >= 2: times.append(e0.elapsed_time(e1))
    res.setdefault(kind, []).append(round(min(times), 3))
if rank == 0:
    print(json.dumps({"gemm_ms_with_concurrent": res, "gemm_tflops_alone": round(2 * M * N * K / min(res["none"]) / 1e9, 1)}))
comm.close(); dist.barrier(); dist.destroy_process_group()
