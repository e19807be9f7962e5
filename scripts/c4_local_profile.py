"""C4 conv stack partitioned for N devices, all partitions on one GPU (loopback
collectives) -- for per-kernel launch lists of the halo-exchange path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import partition, propagate
from paper_2105_04663_b200.executor import Executor
from paper_2105_04663_b200.ir import DType
from paper_2105_04663_b200.workloads import conv_stack
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g, _ = conv_stack((n,), (-1, 0, -1, -1), N=8 // n, H=1024, W=1024, C=128, layers=2,
                  dtype=DType.BF16, with_inputs=False)
ann, _ = propagate(g)
prog = partition(ann, n, plan="fast")
for ins in prog.graph.instructions:
    print(ins.id, ins.opcode.value, ins.shape, file=sys.stderr)
ex = Executor(prog, nparts=n, fuse=True)
ins = [torch.randn((n,) + p.shape.dims, device="cuda").bfloat16() for p in prog.graph.parameters]
for _ in range(2):
    ex.run(ins)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ex.run(ins)
e1.record()
torch.cuda.synchronize()
print("ms", e0.elapsed_time(e1))
