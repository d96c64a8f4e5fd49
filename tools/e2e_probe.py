"""e2e breakdown at C2: H2D of A, b from pinned host + setup + 5 outer steps + D2H of z,
serial copies vs per-node copy stream with ready events (bicadmm_block.ready_event).
python tools/e2e_probe.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg  # noqa: E402

N, M_I, NN, KAPPA = 4, 25_000, 10_000, 100
P = dg.generate(N, M_I, NN, KAPPA, "logistic", seed=1000, device="cuda")
hostA = [a.cpu().pin_memory() for a in P.A]
hostb = [b.cpu().pin_memory() for b in P.b]
del P
torch.cuda.empty_cache()
cs = dg.block_partition(NN, 1)
prm = bc.Params(kappa=KAPPA, max_outer=10 ** 6, inner_fixed=10, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
st = torch.cuda.current_stream()


def run(mode):
    torch.cuda.synchronize()
    E = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    E[0].record(st)
    t0 = time.time()
    if mode == "serial":
        dA = [a.to("cuda", non_blocking=True) for a in hostA]
        db = [b.to("cuda", non_blocking=True) for b in hostb]
        evs = [None] * N
        E[1].record(st)
    else:
        cps = torch.cuda.Stream()
        cps.wait_stream(st)
        dA, db, evs = [], [], []
        with torch.cuda.stream(cps):
            for k in range(N):
                dA.append(hostA[k].to("cuda", non_blocking=True))
                db.append(hostb[k].to("cuda", non_blocking=True))
                ev = torch.cuda.Event()
                ev.record(cps)
                evs.append(ev)
            E[1].record(cps)
        for t_ in dA + db:
            t_.record_stream(st)
    t1 = time.time()
    blocks = [(k, 0, dA[k], evs[k]) if evs[k] is not None else (k, 0, dA[k]) for k in range(N)]
    s = bc.BiCADMM(None, db, "logistic", prm, cs, blocks=blocks)
    t2 = time.time()
    E[2].record(st)
    for _ in range(5):
        s.iterate(1)
    z = s.z
    E[3].record(st)
    torch.cuda.synchronize()
    s.close()
    del s, dA, db
    torch.cuda.empty_cache()
    return dict(mode=mode, total=E[0].elapsed_time(E[3]), h2d=E[0].elapsed_time(E[1]),
                to_setup_end=E[0].elapsed_time(E[2]), steps=E[2].elapsed_time(E[3]),
                host_issue_ms=(t1 - t0) * 1e3, host_setup_ms=(t2 - t1) * 1e3)


for rep in range(3):
    for mode in ("serial", "stream"):
        r = run(mode)
        print({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}, flush=True)
