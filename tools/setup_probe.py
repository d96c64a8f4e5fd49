"""Setup (Gram + factor) device time for the C2 shape: 4 blocks of 25,000 x 10,000 FP64."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg
P = dg.generate(4, 25000, 10000, 100, "logistic", seed=1000, device="cuda")
cs = dg.block_partition(10000, 1)
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s = bc.BiCADMM(P.A, P.b, "logistic", bc.Params(kappa=100, inner_fixed=10), cs)
    e1.record()
    torch.cuda.synchronize()
    print(f"setup {e0.elapsed_time(e1):.1f} ms", flush=True)
    s.close()
