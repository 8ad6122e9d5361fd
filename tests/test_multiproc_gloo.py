"""World-size-2 CPU (gloo) tests of the multi-process protocol of the hot path.

Each rank takes its slice from the C-ABI partitioner (identical on every
rank), computes its partition with the oracle's kernels (Offset trait for
global keys), and the ranks exchange exactly what libmarrow exchanges over
NCCL: hysteresis halo rows + loop-condition all-reduce, MapReduce partial
merge "+" (and max / min for the device reduction stage), N-body COPY re-replication, rebalancer timing all-gather.  The
gathered result must equal the single-partition oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_rows(local, rows_per_rank, shape_tail, dtype):
    """all_gather of variable-length row blocks (pad to the max)."""
    mx = max(rows_per_rank)
    buf = np.zeros((mx,) + shape_tail, dtype=dtype)
    buf[:local.shape[0]] = local
    t = torch.from_numpy(buf.view(np.uint8).copy())
    out = [torch.empty_like(t) for _ in range(WORLD)]
    dist.all_gather(out, t)
    parts = [o.numpy().view(dtype).reshape((mx,) + shape_tail)[:n] for o, n in zip(out, rows_per_rank)]
    return np.concatenate(parts)


def _worker(rank, port, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    from oracle import balance as B
    from oracle import kernels as K
    from paper_1510_06585_b200 import marrow as M

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    out = {}
    d = [0.6, 0.4]
    # ---- Filter pipeline: row partitions, no exchange
    H, W = 37, 50
    off, ln = M.mw_partition_plan(H, 1, d)
    img = synth.np_rgba(3, off[rank] * W, ln[rank] * W).reshape(ln[rank], W, 4)
    mine = K.mirror(K.solarize(K.gauss_noise(img, 4, 8, y0=off[rank]), 128))
    full = _gather_rows(mine, ln, (W, 4), np.uint8)
    whole = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    out["filter"] = np.array_equal(full, K.mirror(K.solarize(K.gauss_noise(whole, 4, 8), 128)))

    # ---- MapReduce: chunk-granule partitions, merge "+" across ranks
    n = 5 * (1 << 16) + 321
    off, ln = M.mw_partition_plan(n, 1 << 16, d)
    x = synth.np_f32_um11(5, off[rank], ln[rank])
    t = torch.tensor([K.sum_(x)], dtype=torch.float64)
    dist.all_reduce(t)
    xs = synth.np_f32_um11(5, 0, n)
    out["mapreduce"] = abs(t.item() - K.sum_(xs)) <= 1e-12 * K.abs_sum(xs)
    # device reduction stage max / min (NEXT-4, R28): partials merged with the
    # same operator (libmarrow: NCCL max / min) equal the whole-domain fold
    y = synth.np_f32_um11(6, off[rank], ln[rank])
    ys = synth.np_f32_um11(6, 0, n)
    ok = True
    for is_min, op in ((False, dist.ReduceOp.MAX), (True, dist.ReduceOp.MIN)):
        t = torch.tensor([K.fold_extreme(x, y, is_min)], dtype=torch.float64)
        dist.all_reduce(t, op=op)
        ok &= t.item() == K.fold_extreme(xs, ys, is_min)
    out["mapreduce_extremes"] = ok

    # ---- Hysteresis: halo rows + loop condition all-reduce (Jacobi per partition)
    H, W = 29, 31
    gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
    L = K.segment(gray, 150, 240)
    off, ln = M.mw_partition_plan(H, 1, d)
    o, m = off[rank], ln[rank]
    cur = L[o:o + m].copy()
    peer = 1 - rank
    e, changed = 0, True
    while changed:
        # halo exchange: rank 0 owns the top rows, rank 1 the bottom rows
        send = torch.from_numpy((cur[-1] if rank == 0 else cur[0]).copy())
        recv = torch.empty(W, dtype=torch.uint8)
        reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
        for r in reqs:
            r.wait()
        halo = recv.numpy()
        ext = np.vstack([cur, halo]) if rank == 0 else np.vstack([halo, cur])
        nxt, ch = K.hyst_step(ext)
        nxt = nxt[:m] if rank == 0 else nxt[1:]
        ch = bool((nxt != cur).any())
        cur = nxt
        flag = torch.tensor([int(ch)])
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)          # loop condition
        changed = bool(flag.item())
        e += 1
    full = _gather_rows(cur, ln, (W,), np.uint8)
    fixed, D = K.hyst_bfs(L)
    out["hysteresis"] = np.array_equal(full, fixed) and e == D + 1

    # ---- N-body: body partitions, COPY re-replication after the step
    N = 600
    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -9)
    off, ln = M.mw_partition_plan(N, 256, d)
    po, vo, _ = K.nbody_step(pos, vel, 1e-4, 1e-3)   # oracle per body is independent
    mine = po[off[rank]:off[rank] + ln[rank]]
    full = _gather_rows(mine, ln, (4,), np.float32)
    out["nbody"] = np.array_equal(full, po)

    # ---- Rebalancer: times all-gathered, identical decision on every rank
    rate = [1.0, 0.25]
    st, p = M.mw_balance_state(), M.mw_balance_defaults()
    dd = [0.5, 0.5]
    decisions = []
    for run in range(4):
        off, ln = M.mw_partition_plan(1 << 20, 256, dd)
        my_t = torch.tensor([ln[rank] / rate[rank] * 1e-6], dtype=torch.float32)
        allt = [torch.empty(1, dtype=torch.float32) for _ in range(WORLD)]
        dist.all_gather(allt, my_t)
        times = [float(a.item()) for a in allt]
        dd, trig = M.mw_balance_step(p, st, times, ln, dd)
        decisions.append((tuple(dd), trig))
    # the oracle takes the same decisions
    so, po_ = B.State(), B.Params()
    od = [0.5, 0.5]
    for run in range(4):
        _, ln = M.mw_partition_plan(1 << 20, 256, od)
        times = [float(np.float32(ln[i] / rate[i] * 1e-6)) for i in range(2)]
        od, ot = B.step(po_, so, times, ln, od)
        if (tuple(od), ot) != decisions[run]:
            out["rebalance"] = False
    out.setdefault("rebalance", decisions[2][1] and not decisions[1][1])
    obj = [decisions]
    dist.broadcast_object_list(obj, src=0)
    out["rebalance_same_on_ranks"] = obj[0] == decisions
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_protocol_gloo():
    port = _port()
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(port, results), nprocs=WORLD, join=True)
    for r in range(WORLD):
        res = dict(results[r])
        assert all(res.values()), (r, res)
