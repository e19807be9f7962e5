"""Copy-engine peer traffic alone vs under a concurrent tcgen05 GEMM on both
ranks (2 ranks): local copy, pull (read the peer's buffer), push (write into
the peer's buffer).  Buffers shared with CUDA IPC (cuda-python)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from cuda.bindings import runtime as rt
from paper_2105_04663_b200 import _capi as C
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
lib = C.lib()
NB = 256 << 20
M, N, K = 8192, 32768, 8192
a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
b = torch.randn(K, N, device=dev, dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
main = torch.cuda.current_stream(); side = torch.cuda.Stream(device=dev)
# IPC-shared region: cudaMalloc directly so the handle covers it exactly
err, base = rt.cudaMalloc(2 * NB)
assert err == 0
err, h = rt.cudaIpcGetMemHandle(base)
handles = [None] * world
dist.all_gather_object(handles, bytes(h.reserved))
peer = {}
for q in range(world):
    if q != rank:
        hh = rt.cudaIpcMemHandle_t(); hh.reserved = handles[q]
        err, p = rt.cudaIpcOpenMemHandle(hh, rt.cudaIpcMemLazyEnablePeerAccess)
        assert err == 0, err
        peer[q] = int(p)
base = int(base)
loc = torch.empty(NB // 2, device=dev, dtype=torch.bfloat16)
other = (rank + 1) % world
D2D = rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice
def copy(kind):
    s = side.cuda_stream
    if kind == "local":
        rt.cudaMemcpyAsync(base + NB, loc.data_ptr(), NB, D2D, s)
    elif kind == "pull":
        rt.cudaMemcpyAsync(loc.data_ptr(), peer[other], NB, D2D, s)
    elif kind == "push":
        rt.cudaMemcpyAsync(peer[other] + NB, loc.data_ptr(), NB, D2D, s)
    elif kind == "push_split4":
        for k in range(4):
            rt.cudaMemcpyAsync(peer[other] + NB + k * NB // 4, loc.data_ptr() + k * NB // 4, NB // 4, D2D, s)
def gemm(n):
    for _ in range(n):
        C.check(lib.spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, main.cuda_stream), "g")
res = []
for kind in ["local", "pull", "push", "push_split4"]:
    for concurrent in (False, True):
        gt, mt = [], []
        for it in range(5):
            torch.cuda.synchronize(); dist.barrier()
            side.wait_stream(main)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(main); s0.record(side)
            copy(kind)
            s1.record(side)
            if concurrent:
                gemm(4)
            m1.record(main)
            main.wait_stream(side)
            torch.cuda.synchronize()
            if it >= 2:
                gt.append(s0.elapsed_time(s1)); mt.append(m0.elapsed_time(m1))
        g = min(gt)
        res.append({"kind": kind, "with_gemm": concurrent, "copy_ms": round(g, 3),
                    "gbs": round(NB / g / 1e6, 1), "gemm4_ms": round(min(mt), 3) if concurrent else None})
if rank == 0:
    for r in res:
        print(json.dumps(r))
torch.cuda.synchronize(); dist.barrier()
for p in peer.values():
    rt.cudaIpcCloseMemHandle(p)
dist.destroy_process_group()
