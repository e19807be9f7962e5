"""Peer all-gather throughput alone vs under a concurrent tcgen05 GEMM on
both ranks (2 or 4 ranks): copy engine (engine 0), background SM pull
(engine 3), SM pull (engine 1), NCCL.  Side-stream events time the gather."""
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
E = int(os.environ.get("GATHER_MB", "256")) << 19          # bf16 elements per rank
comm.ensure_peer(world * E * 2 + (16 << 20), dev)
M, N, K = 8192, 32768, 8192
a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
b = torch.randn(K, N, device=dev, dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
main = torch.cuda.current_stream(); side = torch.cuda.Stream(device=dev)
src = torch.randn(E, device=dev, dtype=torch.bfloat16)
dst = torch.empty(world * E, device=dev, dtype=torch.bfloat16)
garr, ng, gs = _groups_arg([list(range(world))])
sh_in, sh_out = Shape((E,), DType.BF16), Shape((world * E,), DType.BF16)
def gemm(n):
    for _ in range(n):
        C.check(lib.spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, main.cuda_stream), "g")
def gather(kind):
    with torch.cuda.stream(side):
        if kind == "nccl":
            dist.all_gather_into_tensor(dst, src)
        else:
            eng = {"ce": 0, "sm": 1, "sm_bg": 3}[kind]
            C.check(lib.spmd_peer_all_gather(comm.handle, desc(src.view(1, -1), sh_in), desc(dst.view(1, -1), sh_out),
                                             0, garr, ng, gs, 0, 1, eng, side.cuda_stream), "ag")
res = []
sms = torch.cuda.get_device_properties(dev).multi_processor_count
for reserve in [int(x) for x in os.environ.get("GEMM_RESERVE", "0").split(",")]:
  lib.spmd_set_sm_limit(sms - reserve if reserve else 0)
  for kind in os.environ.get("GATHER_KINDS", "ce,sm_bg,sm,nccl").split(","):
    for concurrent in (False, True):
        gt, mt = [], []
        for it in range(5):
            torch.cuda.synchronize(); dist.barrier()
            side.wait_stream(main)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(main)
            s0.record(side)
            gather(kind)
            s1.record(side)
            if concurrent:
                gemm(4)
            m1.record(main)
            main.wait_stream(side)
            torch.cuda.synchronize()
            if it >= 2:
                gt.append(s0.elapsed_time(s1)); mt.append(m0.elapsed_time(m1))
        g = min(gt)
        res.append({"reserve": reserve, "kind": kind, "with_gemm": concurrent, "gather_ms": round(g, 3),
                    "recv_gbs": round((world - 1) * E * 2 / g / 1e6, 1),
                    "gemm4_ms": round(min(mt), 3) if concurrent else None})
if rank == 0:
    for r in res:
        print(json.dumps(r))
comm.close(); dist.barrier(); dist.destroy_process_group()
