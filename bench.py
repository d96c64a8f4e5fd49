#!/usr/bin/env python
"""Benchmark of the Bi-cADMM hot path on B200 (one JSON line on rank 0).

Metric (BASELINE.json): Bi-cADMM inner iterations/s (+ GEMV HBM GB/s vs peak).
Unit: node-level inner iterations per second -- one Algorithm-2 sharing-ADMM
sweep (Eqs. (22)-(24): GEMV-T, H-apply, GEMV, block sum, prox, dual update) of
one node's local problem, summed over all nodes of the job.

Workload (N=1): configs[1], sparse logistic regression, 4 nodes x m_i = 25,000
samples (m = 100k), n = 10,000 features, kappa = 100, one feature block per node
(M = 1), FP64.  A "step" is one outer Bi-cADMM iteration: K_in = 10 inner sweeps
on every node, then the global step (Collect, (7b), (13), (14), (9), (15)) and
the per-iteration residual read-back.  Inputs (8 GB of A) exceed the 126 MB L2,
so no flush is needed between steps.

Multi-GPU (torchrun, N > 1): weak scaling -- every rank holds 4 more nodes of the
same shape (node-major placement: no per-sweep exchange); the consensus step
all-reduces the n-vector sum_i (x_i + u_i) and the node residuals over NCCL.

--impl reference: the FP64 CPU oracle (oracle/, test infrastructure) timed as it
stands on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Bi-cADMM inner iters/sec and time-to-tol at 1/2/4/8 B200; GEMV HBM GB/s vs peak"
UNIT = "inner_iters/s"
WORKLOAD = ("configs[1]: sparse logistic regression, N=4 nodes x m_i=25000 (m=100k), n=10000, kappa=100, "
            "M=1 feature block per node, FP64, K_in=10 inner sweeps per outer step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="ranks (one per GPU); without a torchrun environment bench.py launches them itself")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--inner", type=int, default=10)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--nodes", type=int, default=4, help="nodes per rank (node placement) / in total (block)")
    ap.add_argument("--m", type=int, default=25_000)
    ap.add_argument("--n", type=int, default=10_000)
    ap.add_argument("--kappa", type=int, default=100)
    ap.add_argument("--loss", default="logistic")
    ap.add_argument("--placement", default=None, choices=["node", "block"],
                    help="node-major (weak scaling, whole nodes per rank) or block-major (feature blocks "
                         "over the ranks, Algorithm 2's per-sweep AllReduce); default from --config")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-max-gb", type=float, default=24.0,
                    help="skip the e2e pass (pinned host copy of A) when a rank's A exceeds this")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-m", type=int, default=25_000, help="cpu_baseline sample rows (default: a full node)")
    ap.add_argument("--cpu-n", type=int, default=10_000, help="cpu_baseline sample columns (default: a full node)")
    ap.add_argument("--cpu-sweeps", type=int, default=10, help="oracle inner sweeps timed for cpu_baseline")
    ap.add_argument("--sweep", type=int, default=0, help="0 auto (fused single pass), 1 two-pass, 2 fused")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance rows")
    ap.add_argument("--ttt-max-outer", type=int, default=1000,
                    help="cap of the configs[1] time-to-tolerance solve (outer iterations)")
    ap.add_argument("--no-prof", action="store_true",
                    help="no per-phase events in the timed region (launch-overhead study; roofline null)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the ranks and print each rank's placement (no GPU work); launcher check")
    ap.add_argument("--config", default="C2", choices=sorted(PRESETS),
                    help="BASELINE.json config preset; C2 = configs[1] (default)")
    pre, _ = ap.parse_known_args()
    pr = PRESETS[pre.config]
    ap.set_defaults(**{k: v for k, v in pr.items() if k not in ("workload", "placement")})   # flags still win
    a = ap.parse_args()
    if a.placement is None:
        a.placement = pr.get("placement", "node")
    a.workload = pr["workload"]
    if a.dtype == "f32":   # the presets name the paper's FP64 arithmetic; say what this run stores
        a.workload = a.workload.replace("FP64", "FP32 storage")
    if a.config == "C3w":   # weak scaling W3: one 12,500-column block per GPU
        G = int(os.environ.get("WORLD_SIZE", a.gpus))
        a.n, a.M, a.kappa = 12_500 * G, G, 125 * G
    return a


# Shapes of BASELINE.json configs.  placement "node": per-rank shape
# (weak scaling over ranks); "block": the whole problem, feature blocks spread over the ranks.
PRESETS = {
    "C2": dict(nodes=4, m=25_000, n=10_000, kappa=100, loss="logistic", C=1, M=1, inner=10, workload=WORKLOAD),
    "C2ls": dict(nodes=4, m=25_000, n=10_000, kappa=100, loss="ls", C=1, M=1, inner=10,
                 workload="configs[1] shape with the LS loss (diagnostic: closed-form prox)"),
    "C1": dict(nodes=2, m=100, n=50, kappa=5, loss="ls", C=1, M=1, inner=10,
               workload="configs[0]: sparse LS, N=2 nodes x m_i=100, n=50, kappa=5, M=1, FP64 (launch-bound)"),
    "C3": dict(nodes=1, m=1_000_000, n=100_000, kappa=1000, loss="ls", C=1, M=8, inner=5, placement="block",
               workload="configs[2]: sparse LS, m=1M, n=100k, kappa=1000, 8 feature blocks over the GPUs "
                        "(block-major; FP64 needs 8 GPUs: 100 GB of A each), K_in=5"),
    "C3w": dict(nodes=1, m=1_000_000, n=12_500, kappa=125, loss="ls", C=1, M=1, inner=5, placement="block",
                workload="configs[2] weak scaling (SURVEY 8(d) W3): sparse LS, m=1M, one n_j=12,500 feature "
                         "block per GPU (n = 12,500 G, kappa = 125 G), K_in=5"),
    "C4": dict(nodes=1, m=500_000, n=20_000, kappa=500, loss="softmax", C=10, M=8, inner=5, placement="block",
               workload="configs[3]: sparse softmax, C=10 classes, N=1 node x m=500k, n=20k, kappa=500, "
                        "M=8 feature blocks over the GPUs (block-major, strong scaling), FP64, K_in=5 "
                        "(A = 80 GB in total)"),
    "C5": dict(nodes=8, m=250_000, n=50_000, kappa=1000, loss="hinge", C=1, M=8, inner=5, placement="block",
               workload="configs[4]: sparse hinge SVM, 8 nodes x m_i=250k, n=50k, kappa=1000, 8 feature blocks "
                        "(block-major: GPU g holds block g of every node; FP64 needs 8 GPUs), K_in=5"),
    "C5s": dict(nodes=8, m=250_000, n=6_250, kappa=125, loss="hinge", C=1, M=1, inner=5,
                workload="configs[4] per-GPU shard stand-in (one block of each of the 8 nodes as M=1 nodes: "
                         "no block-sum AllReduce), sparse hinge, m_i=250k x n_j=6,250, FP64, K_in=5 (A = 100 GB)"),
    "C3s": dict(nodes=1, m=1_000_000, n=12_500, kappa=125, loss="ls", C=1, M=1, inner=5,
                workload="configs[2] per-GPU shard stand-in (one of the 8 feature blocks as an M=1 node: no "
                         "block-sum AllReduce), sparse LS, m=1M x n_j=12.5k, FP64, K_in=5 (A = 100 GB)"),
}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.dev = device_index

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except Exception:
                continue
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle timing
def oracle_sample(m: int, n_s: int, inner: int, outer: int, warmup: int, n_full: int, m_full: int, seed=7):
    """Time the oracle's Algorithm-2 sweeps on ONE node of m rows x n_s columns of the
    bench distribution (logistic, M = 1): `warmup` + `outer` outer iterations of `inner`
    sweeps; the timed figure is the wall time of the last `outer` outer iterations (the
    oracle's per-iteration clock, orc_result.step_s).  Its setup (Gram + Cholesky) is
    reported separately.  By default the sample IS a full C2 node (25,000 x 10,000), so
    no scaling is applied; a smaller sample is scaled by the per-sweep algorithmic-byte
    ratio and flagged `extrapolated`."""
    from oracle import oracle as orc
    from paper_2405_16267_b200 import datagen as dg
    import numpy as np
    kappa = max(1, n_s // 100)
    P = dg.generate(1, m, n_s, kappa, "logistic", seed=seed)
    pb = orc.Problem([P.A[0].numpy()], [P.b[0].numpy()], orc.LOGISTIC, 1, np.array([0, n_s]))
    del P
    total = warmup + outer
    t0 = time.time()
    r = orc.run(pb, orc.Params(kappa=kappa, max_outer=total, inner_fixed=inner, refit=0,
                               eps_p=0, eps_d=0, eps_b=0))
    wall = time.time() - t0
    step_s = r["step_s"][warmup:total]
    sweeps = outer * inner
    per_sweep_s = float(np.sum(step_s)) / sweeps
    bytes_sample = 8 * (2 * m * n_s + n_s * n_s)
    bytes_full = 8 * (2 * m_full * n_full + n_full * n_full)
    scale = bytes_full / bytes_sample
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    what = "a full configs[1] node" if scale == 1.0 else f"scaled by the algorithmic-byte ratio {scale:.2f}"
    return dict(value=1.0 / per_sweep_s / scale, scale=scale, cores=cores, setup_s=r["timings"]["setup_s"],
                per_sweep_s=per_sweep_s, step_s=[float(x) for x in step_s], wall_s=wall,
                sample=f"oracle (FP64 C, OpenMP over {cores} host threads): 1 node, m_i={m} x n={n_s} logistic "
                       f"({what}); {outer} outer step(s) x K_in={inner} sweeps timed after {warmup} untimed; "
                       f"setup (Gram + Cholesky, {r['timings']['setup_s']:.1f} s) excluded")


# ----------------------------------------------------------------------------- launch
def maybe_spawn(args) -> bool:
    """--gpus N without a torchrun environment: re-launch this command as N ranks
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1).  Returns True
    when the ranks ran here (the caller exits with their status)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
        return False
    if args.gpus <= 1:
        return False
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    sys.exit(rc)


# ----------------------------------------------------------------------------- our arm
def local_problem(args, world, rank, local, dist, bc, dg, torch):
    """This rank's blocks and labels.

    node placement (weak scaling): every rank holds `nodes` whole nodes (M blocks each),
    drawn by datagen.generate with seed 1000 + rank; Algorithm 2's block sums stay local.
    block placement: placement.plan(world, N, M, "block") gives rank g the
    block group g of every node; the blocks are drawn one by one (datagen.generate_blocks),
    the labels' partial products summed over the ranks by a torch.distributed all-reduce
    (data preparation, outside the timed region)."""
    from paper_2405_16267_b200 import placement as pl
    dtype = torch.float64 if args.dtype == "f64" else torch.float32
    n, m, C, M = args.n, args.m, args.C, args.M
    cs = dg.block_partition(n, M, align=int(os.environ.get("BENCH_BLOCK_ALIGN", "16")))
    if args.placement == "node":
        nl = args.nodes
        N = nl * world
        P = dg.generate(nl, m, n, args.kappa, args.loss, C=C, seed=1000 + rank, device="cuda", dtype=dtype)
        if n % 4:   # rows must start 16-byte aligned (lda % 4 == 0): pad the node matrices, one at a time
            for k in range(len(P.A)):
                t = torch.zeros(P.A[k].shape[0], -(-n // 4) * 4, dtype=P.A[k].dtype, device=P.A[k].device)
                t[:, :n] = P.A[k]
                P.A[k] = t
                del t
                torch.cuda.empty_cache()
        b_all = [None] * N
        blocks = []
        for k in range(nl):
            i = rank * nl + k
            b_all[i] = P.b[k]
            for j in range(M):
                blocks.append((i, j, P.A[k][:, cs[j]:cs[j + 1]]))
        color = rank
        del P
    else:
        N = args.nodes
        plans = pl.plan(world, N, M, "block")
        pl.check(plans, N, M)
        me = plans[rank]

        def allsum(plist):
            if world > 1:
                for t in plist:
                    dist.all_reduce(t)

        A, b_all, _ = dg.generate_blocks(N, m, n, args.kappa, args.loss, cs, me.blocks, C=C, seed=1000,
                                         device="cuda", dtype=dtype, sum_products=allsum)
        blocks = [(i, j, A[(i, j)]) for (i, j) in me.blocks]
        color = me.node_group
    torch.cuda.empty_cache()
    return N, cs, b_all, blocks, color


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2405_16267_b200 import bicadmm as bc
    from paper_2405_16267_b200 import datagen as dg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, m, C, M = args.n, args.m, args.C, args.M
    N, cs, b_all, blocks, color = local_problem(args, world, rank, local, dist, bc, dg, torch)
    local_nodes = sorted({i for i, _, _ in blocks})
    comm = None
    if world > 1:
        uid = [bc.bicadmm_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = bc.bicadmm_comm_init(world, rank, local, uid[0], color)
    elif os.environ.get("BICADMM_NCCL_SELF"):   # one-rank NCCL communicator: the multi-rank code path
        comm = bc.bicadmm_comm_init(1, 0, local, None, 0)
    prm = bc.Params(kappa=args.kappa, max_outer=10 ** 6, inner_fixed=args.inner, refit=0,
                    eps_p=0.0, eps_d=0.0, eps_b=0.0, sweep=args.sweep)
    t0 = time.time()
    solver = bc.BiCADMM(None, b_all, args.loss, prm, cs, blocks=blocks, comm=comm, C=C)
    setup_wall = time.time() - t0
    kind = solver.sweep_kind()[0]
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        solver.iterate(1)
    # per-phase CUDA events inside the timed region (the roofline's live kernel times) cost
    # ~1 % at configs[1]; at the launch-bound configs[0] they also disable the CUDA-graph replay
    # (3.3x), so there the timed region runs without them and a second, profiled pass of the
    # same K steps supplies the kernel table
    prof_in_timed = not args.no_prof and args.config != "C1"
    solver.set_profiling(prof_in_timed)
    launches0 = solver.launches()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        solver.iterate(1)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    launches = solver.launches() - launches0
    if not prof_in_timed and not args.no_prof:   # the separate profiled pass (configs[0])
        solver.set_profiling(True)
        for _ in range(args.steps):
            solver.iterate(1)
        torch.cuda.synchronize()
    phases = solver.phases()
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    sweeps = args.steps * args.inner
    value = N * sweeps / (ms / 1e3)
    sc = solver.scalars()

    # roofline of the dominant kernel (one HBM pass over every local A_ij)
    def h_bytes(nj, s, C):
        # C == 1 (default): packed lower 64x64 tiles of H (k_symv.cu) + x, y; C > 1: full H
        if C == 1 and os.environ.get("BICADMM_HPACK", "1") != "0":
            nb = (nj + 63) // 64
            return nb * (nb + 1) // 2 * 4096 * s + 16 * nj
        return nj * nj * s + 16 * C * nj

    s = 8 if args.dtype == "f64" else 4
    shapes = [(a.shape[0], a.shape[1]) for _, _, a in blocks]
    A_bytes = sum(r * c for r, c in shapes) * s
    byt = {"gemv": A_bytes + sum(8 * C * (c + r) for r, c in shapes),
           "gemv_t_partial": A_bytes + sum(16 * C * r for r, c in shapes),
           "h_apply": sum(h_bytes(c, s, C) for r, c in shapes),
           # fused: A once from HBM + x and the per-sample vectors b, p, nu, delta, omega
           "fused_sweep": A_bytes + len(local_nodes) * (8 * n * C + s * m + 8 * 5 * m * C)}
    # per-sweep phases are timed per call (one call = one sweep; the packed H-apply is
    # two kernels per call: tiles + fixed-order reduce)
    per_sweep = ("gemv_t_partial", "gemv_t_reduce", "h_apply", "gemv", "prox", "fused_sweep", "allreduce")

    def calls(k, v):
        return sweeps if (k in per_sweep and v[1] > 0) else v[1]

    cand = {k: phases[k] for k in byt if phases[k][1] > 0}
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    dom, achieved = None, None
    if cand:   # absent with --no-prof
        dom = max(cand, key=lambda k: cand[k][0])
        dms, dcnt = cand[dom]
        avg_s = dms / calls(dom, cand[dom]) / 1e3
        achieved = byt[dom] / avg_s / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        key = args.config if args.dtype == "f64" else f"{args.config}/{args.dtype}"
        traffic = tr.get(key, {}).get(dom, {}).get("bytes_per_launch")
    except Exception:
        pass
    total_phase = sum(v[0] for v in phases.values())
    kernels = {k: {"ms_per_call": (v[0] / calls(k, v) if v[1] else None), "launches": v[1],
                   "calls": calls(k, v), "share": v[0] / total_phase if total_phase else None,
                   **({"GB_per_s": byt[k] / (v[0] / calls(k, v) / 1e3) / 1e9} if k in byt and v[1] else {})}
               for k, v in phases.items()}
    solver.close()
    del solver

    # e2e: through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if args.no_e2e:
        e2e = None
    elif A_bytes > args.e2e_max_gb * 1e9:
        e2e = {"value": None, "unit": UNIT, "skipped": f"local A is {A_bytes / 1e9:.0f} GB (> --e2e-max-gb "
               f"{args.e2e_max_gb}): no pinned host copy of it on this box"}
    else:
        def host_copy(a):   # pinned, rows padded to a 16-byte multiple (lda % 4 == 0, as on the device)
            w = -(-a.shape[1] // 4) * 4
            t = torch.zeros(a.shape[0], w, dtype=a.dtype).pin_memory()
            t[:, :a.shape[1]] = a.cpu()
            return t

        hostA = [host_copy(a) for _, _, a in blocks]
        widths = [a.shape[1] for _, _, a in blocks]
        hostb = {i: b_all[i].cpu().pin_memory() for i in local_nodes}
        block_ids = [(i, j) for i, j, _ in blocks]
        del blocks, b_all
        torch.cuda.empty_cache()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        cps = torch.cuda.Stream()

        def e2e_once():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            # block k's H2D on a copy stream, one ready event per block: setup's Gram of block k
            # waits on its own event only (bicadmm_block.ready_event), so later copies overlap
            # earlier Grams
            cps.wait_stream(stream)
            db, dA, evs = {}, [], []
            with torch.cuda.stream(cps):
                for i in local_nodes:
                    db[i] = hostb[i].to("cuda", non_blocking=True)
                for k in range(len(hostA)):
                    dA.append(hostA[k].to("cuda", non_blocking=True))
                    ev = torch.cuda.Event()
                    ev.record(cps)
                    evs.append(ev)
            for t_ in dA + list(db.values()):
                t_.record_stream(stream)
            b2 = [db.get(i) for i in range(N)]
            blocks2 = [(ij[0], ij[1], dA[k][:, :widths[k]], evs[k]) for k, ij in enumerate(block_ids)]
            s2 = bc.BiCADMM(None, b2, args.loss, prm, cs, blocks=blocks2, comm=comm, C=C)
            for _ in range(args.steps):
                s2.iterate(1)          # each step reads back its 6 residual scalars
            z = s2.z                   # D2H of the result
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ems], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ems = float(t.item())
            s2.close()
            return ems, z

        e2e_once()                 # untimed warm-up pass (first-use costs of the copy stream)
        if world > 1:
            dist.barrier()
        ems, z = e2e_once()
        h2d = sum(a.numel() * a.element_size() for a in hostA) + sum(b.numel() * b.element_size()
                                                                    for b in hostb.values())
        e2e = {"value": N * sweeps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d / args.steps),
               "d2h_bytes_per_step": int((6 * 8 * args.steps + z.nbytes) / args.steps),
               "ms_total": ems, "includes": "H2D of A, b (per-block copy stream, overlapping setup's Gram) + "
                                            "setup (Gram+factor) + steps + D2H of z; second of two passes"}

    ttt = None
    if rank == 0 and world == 1 and not args.no_ttt and args.config == "C2":
        ttt = {"configs[1]": time_to_tol_c2(bc, dg, np, torch, args),
               "table1": time_to_tol(bc, dg, np, torch, args.sweep)}
    if rank == 0 and world == 1 and not args.no_ttt and args.config == "C1":
        ttt = {"configs[0]": time_to_tol_c1(bc, dg, np, torch)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == "C2":
        o = oracle_sample(args.cpu_m, args.cpu_n, args.inner, max(1, args.cpu_sweeps // args.inner), 0, n, m)
        cpu = {"value": o["value"], "unit": UNIT, "cores": o["cores"], "kind": "oracle", "sample": o["sample"],
               "setup_s": o["setup_s"], "extrapolated": o["scale"] != 1.0}
        if ttt is not None:   # the oracle's time-to-tol at configs[1] is the same outer-iteration count
            ttt["configs[1]"]["oracle_model_s"] = (o["setup_s"] * 4 + ttt["configs[1]"]["inner_sweeps"] * 4
                                                   * o["per_sweep_s"])
            ttt["configs[1]"]["oracle_model"] = ("modelled, not run: 4 x oracle setup + (GPU outer iterations x "
                                                 "K_in x 4 nodes) x the oracle's measured per-sweep time (the "
                                                 "iterates agree to 1e-9, so the oracle stops at the same outer "
                                                 "iteration)")

    if rank == 0:
        scaling = "weak" if args.placement == "node" or args.config == "C3w" else "strong"
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded, P:268 recipe; DESIGN.md 5)",
            "config": {"workload": args.workload, "preset": args.config, "C": C, "M": M,
                       "nodes_total": N, "local_blocks": len(shapes), "m_i": m, "n": n, "kappa": args.kappa,
                       "K_in": args.inner,
                       "placement": ("single GPU" if world == 1 else "node-major") if args.placement == "node"
                       else f"block-major ({M} feature blocks over {world} GPU(s))",
                       "l2": "inputs larger than L2 (A = %.1f GB/rank)" % (A_bytes / 1e9),
                       "sweeps_per_s": sweeps / (ms / 1e3), "setup_wall_s": setup_wall,
                       "inner_sweep": {4: "fused single HBM pass (k_fused4: CTA-pair clusters, SURVEY 8(f)1)",
                                       5: "whole inner loops in one CTA per node (k_small_sweeps: A_ij, H_ij "
                                          "staged in shared memory once per outer iteration)"}.get(
                                           kind, "two-pass (GEMV-T + H-apply + GEMV)"),
                       "two_pass_equivalent_GBps": (2 * A_bytes + sum(c * c for r, c in shapes) * s) * sweeps
                       / (ms / 1e3) / 1e9},
            "roofline": None if dom is None else {
                "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "timing": "CUDA events inside the timed region" if prof_in_timed else
                          "CUDA events of a second, profiled pass of the same K steps (launch-bound config)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks else "fallback"},
            "kernels": kernels,
            "cpu_baseline": cpu,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": launches,
            "time_to_tol": ttt,
            "residuals_last": sc,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def time_to_tol_c2(bc, dg, np, torch, args):
    """configs[1] to tolerance (SURVEY 8(d) C2 "time-to-tol"): the bench's own data
    (seed 1000), K_in = 10 fixed, p_r, d_r, b_r <= 1e-4 (DESIGN R6); device time of
    setup (Gram + factor) + solve (CUDA-graph while loop, device-side termination)."""
    P = dg.generate(4, 25_000, 10_000, 100, "logistic", seed=1000, device="cuda")
    cs = dg.block_partition(10_000, 1)
    prm = bc.Params(kappa=100, max_outer=args.ttt_max_outer, inner_fixed=10, refit=0, sweep=args.sweep)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s = bc.BiCADMM(P.A, P.b, "logistic", prm, cs)
    e1.record()
    rep = s.solve()
    e2.record()
    torch.cuda.synchronize()
    sup = s.support()
    truth = np.nonzero(P.x_true.cpu().numpy())[0]
    out = {"workload": "configs[1] (4 nodes x 25,000 x 10,000 logistic, kappa=100, FP64), K_in=10, eps=1e-4",
           "s": e0.elapsed_time(e2) / 1e3, "setup_s": e0.elapsed_time(e1) / 1e3, "solve_s": e1.elapsed_time(e2) / 1e3,
           "outer_iters": rep.outer_iters, "inner_sweeps": int(rep.inner_sweeps), "converged": bool(rep.converged),
           "p_r": rep.p_r, "d_r": rep.d_r, "b_r": rep.b_r,
           "support_overlap_with_x_true": int(np.intersect1d(sup, truth).size), "kappa": 100}
    s.close()
    del P
    torch.cuda.empty_cache()
    return out


def time_to_tol_c1(bc, dg, np, torch, seeds=10):
    """configs[0] to tolerance on the GPU and on the oracle ("C1 and C2 run the
    full time-to-tol on the oracle"): 2 nodes x 100 x 50, kappa = 5, K_in = 10, eps = 1e-4;
    GPU device time (CUDA events, setup + solve in a CUDA-graph while loop) against the
    oracle's wall time on the host, same seeds, same outer-iteration count expected."""
    from oracle import oracle as orc
    rows = []
    for seed in range(seeds):
        P = dg.generate(2, 100, 50, 5, "ls", seed=seed)
        cs = dg.block_partition(50, 1)
        prm = dict(kappa=5, max_outer=2000, inner_fixed=10, refit=1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls", bc.Params(**prm), cs)
        rep = s.solve()
        e1.record()
        torch.cuda.synchronize()
        gpu_s = e0.elapsed_time(e1) / 1e3
        sup = s.support()
        s.close()
        t0 = time.time()
        ref = orc.run(orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LS, 1, np.array(cs)),
                      orc.Params(**prm))
        cpu_s = time.time() - t0
        rows.append(dict(seed=seed, gpu_s=gpu_s, oracle_s=cpu_s, outer_gpu=rep.outer_iters, outer_oracle=ref["iters"],
                         converged=bool(rep.converged), same_support=sup.tolist() == ref["support"].tolist()))
    return {"workload": "configs[0]: sparse LS, 2 nodes x 100 x 50, kappa = 5, K_in = 10, eps = 1e-4, LS refit",
            "seeds": seeds, "gpu_s_median": float(np.median([r["gpu_s"] for r in rows])),
            "oracle_s_median": float(np.median([r["oracle_s"] for r in rows])),
            "oracle_cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
            "same_outer_iterations": all(r["outer_gpu"] == r["outer_oracle"] for r in rows),
            "same_support": all(r["same_support"] for r in rows), "runs": rows}


def time_to_tol(bc, dg, np, torch, sweep):
    """Table-1-shaped SLS row: N=4 nodes, m=3e5, n=4000, s_l=0.9 (kappa=400),
    solved to p_r, d_r, b_r <= 1e-4; device time of setup + solve (CUDA events)."""
    n, m, N, sl = 4000, 300_000, 4, 0.9
    kappa = int(round(n * (1 - sl)))
    P = dg.generate(N, m // N, n, kappa, "ls", seed=0, device="cuda")
    cs = dg.block_partition(n, 1)
    prm = bc.Params(kappa=kappa, max_outer=3000, inner_fixed=10, refit=1, sweep=sweep)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s = bc.BiCADMM(P.A, P.b, "ls", prm, cs)
    e1.record()
    rep = s.solve()
    e2.record()
    torch.cuda.synchronize()
    sup = s.support()
    truth = np.nonzero(P.x_true.cpu().numpy())[0]
    out = {"workload": "Table-1 row (P:294): SLS, N=4 nodes, m=3e5, n=4000, s_l=0.9 (kappa=400), FP64, "
                       "eps=1e-4, K_in=10, LS refit",
           "s": e0.elapsed_time(e2) / 1e3, "setup_s": e0.elapsed_time(e1) / 1e3, "solve_s": e1.elapsed_time(e2) / 1e3,
           "outer_iters": rep.outer_iters, "inner_sweeps": int(rep.inner_sweeps), "converged": bool(rep.converged),
           "support_recovered": bool(np.array_equal(np.sort(sup), truth)),
           "paper_s": 4.1, "paper_hw": "i7-13700 + RTX 4070, PsFiT/PyTorch (P:265-267, P:294); context, not target"}
    s.close()
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as it stands on the host cores: each step = one outer iteration of
    K_in sweeps on ONE full configs[1] node (a quarter of our step's 4 nodes; the unit,
    node-level inner iterations/s, is the same).  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    t0 = time.time()
    o = oracle_sample(args.cpu_m, args.cpu_n, args.inner, args.steps, args.warmup, args.n, args.m)
    value = o["value"]
    ms_per_step = args.inner * 1e3 / value
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, args.gpus), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, P:268 recipe)",
        "config": {"workload": args.workload, "preset": args.config, "K_in": args.inner,
                   "step": "one outer iteration (K_in sweeps) of one node"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": o["cores"], "kind": "oracle", "sample": o["sample"],
                         "setup_s": o["setup_s"], "extrapolated": o["scale"] != 1.0},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "ours":
        maybe_spawn(args)
    if args.dry_run:
        from paper_2405_16267_b200 import placement as pl
        world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
        N = args.nodes * world if args.placement == "node" else args.nodes
        me = pl.plan(world, N, args.M, args.placement)[rank]
        time.sleep(0.3 * rank)   # one line per rank, not interleaved
        print(json.dumps({"dry_run": True, "rank": rank, "world": world, "placement": args.placement,
                          "node_group": me.node_group, "blocks": me.blocks}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
