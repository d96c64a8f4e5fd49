import torch, sys
sys.path.insert(0, '.')
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg
P = dg.generate(2, 100, 50, 5, "ls", seed=0)
cs = dg.block_partition(50, 1)
s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls", bc.Params(kappa=5, max_outer=10, inner_fixed=10), cs)
l0 = s.launches()
s.iterate(3)
print("launches", s.launches() - l0, flush=True)
