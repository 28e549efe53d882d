"""CPU, world_size 2 over gloo: the multi-GPU host protocol.

Each rank owns a contiguous shard [r*N/G, (r+1)*N/G) (cupso.shard_range),
advances it one iteration with the iteration-start snapshot, encodes its best
admitted candidate as a cupso record, all-gathers the records, and applies
select_winner -- exactly what libcupso's k_propose / ncclAllGather / k_commit
do on the device. The per-shard step here is the oracle (checker) so the
protocol itself is verified against run_serial without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fitness, n, d, T, seed, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as orc
        from paper_2205_01313_b200.swarm import (decode_record, encode_record, select_winner,
                                                 shard_range)
        o = orc.Oracle()
        p = o.make_params(fitness, n, d, T)
        st, gfit, gidx, gpos = o.init(fitness, n, d, seed)  # replicated init (same Philox)
        first, count = shard_range(n, world, rank)
        trace, tpart = [], []
        for t in range(T):
            bf, bi, bp, adm = o.shard_step(fitness, p, seed, t, st, first, count, gpos, gfit)
            rec = encode_record(bf, bi, adm, bp)
            recs = [None] * world
            dist.all_gather_object(recs, rec)
            dec = [decode_record(r, d) for r in recs]
            w = select_winner([(f, i) for f, i, _, _ in dec], gfit)
            if w >= 0:
                gfit, gidx, gpos = dec[w][0], dec[w][1], dec[w][3]
            trace.append(gfit)
            tpart.append(gidx)
        out_q.put((rank, np.array(trace), np.array(tpart), gpos, sum(x[2] for x in dec)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("sphere", 257, 3, 30, 5), ("cubic", 200, 1, 25, 2),
                                  ("rosenbrock", 101, 4, 20, 8)])
def test_two_rank_exchange_reproduces_serial(oracle, case):
    fitness, n, d, T, seed = case
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fitness, n, d, T, seed, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ref = oracle.run_serial(fitness, n, d, T, seed)
    for rank, trace, tpart, gpos, _ in results:
        assert np.array_equal(trace.view(np.uint64), ref.trace.view(np.uint64)), f"rank {rank}"
        assert np.array_equal(tpart, ref.trace_particle), f"rank {rank}"
        assert np.array_equal(gpos.view(np.uint64), ref.gbest_pos.view(np.uint64)), f"rank {rank}"


# ------------------------------------------------- speculative passes (k_spec)
def _spec_worker(rank, world, port, fitness, n, d, T, seed, kmax, out_q):
    """The sharded speculative protocol of libcupso (k_spec + all-gather of a
    SpecRec per pass + k_spec_commit), restated on CPU: each rank runs K
    iterations of its shard against the fixed snapshot, stops at its first
    admission before the pass's last iteration, all-gathers (tmin, admitted,
    candidate) and applies spec_decide; a falsified pass restores the
    pre-pass state (buffer A) and re-runs [t0, tmin]."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as orc
        from paper_2205_01313_b200.swarm import NO_PARTICLE, shard_range, spec_decide
        o = orc.Oracle()
        p = o.make_params(fitness, n, d, T)
        st, gfit, gidx, gpos = o.init(fitness, n, d, seed)
        first, count = shard_range(n, world, rank)
        trace = np.zeros(T)
        tpart = np.zeros(T, dtype=np.uint32)
        t0, K, kspec, passes, fails = 0, 1, 1, 0, 0
        while t0 < T:
            A = {k: v.copy() for k, v in st.items()}
            tl = t0 + K - 1
            tmin, cand = 0xFFFFFFFF, (0, -np.inf, NO_PARTICLE, np.zeros(d))
            for t in range(t0, t0 + K):
                bf, bi, bp, adm = o.shard_step(fitness, p, seed, t, st, first, count, gpos, gfit)
                if adm and t < tl:
                    tmin = t
                    break
                if t == tl:
                    cand = (adm, bf, bi, bp)
            recs = [None] * world
            dist.all_gather_object(recs, (tmin, cand[0], cand[1], cand[2], cand[3]))
            dec = spec_decide([r[:4] for r in recs], t0, K, kspec, kmax, T)
            passes += 1
            if dec["failed"]:
                fails += 1
                st = A
            else:
                trace[t0:tl] = gfit
                tpart[t0:tl] = gidx
                if dec["winner"] >= 0:
                    w = recs[dec["winner"]]
                    gfit, gidx, gpos = w[2], w[3], w[4]
                trace[tl], tpart[tl] = gfit, gidx
            t0, K, kspec = dec["t0"], dec["K"], dec["kspec"]
        out_q.put((rank, trace, tpart, gpos, passes, fails, st["positions"].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("sphere", 257, 3, 40, 5, 8), ("cubic", 200, 1, 60, 2, 64),
                                  ("rosenbrock", 101, 4, 30, 8, 4)])
def test_two_rank_speculative_passes_reproduce_serial(oracle, case):
    fitness, n, d, T, seed, kmax = case
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spec_worker, args=(r, world, port, fitness, n, d, T, seed, kmax, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ref = oracle.run_serial(fitness, n, d, T, seed)
    from paper_2205_01313_b200.swarm import shard_range
    pos = ref.state["positions"].reshape(d, n)
    for rank, trace, tpart, gpos, passes, fails, mypos in results:
        assert np.array_equal(trace.view(np.uint64), ref.trace.view(np.uint64)), f"rank {rank}"
        assert np.array_equal(tpart, ref.trace_particle), f"rank {rank}"
        assert np.array_equal(gpos.view(np.uint64), ref.gbest_pos.view(np.uint64)), f"rank {rank}"
        first, count = shard_range(n, world, rank)
        got = mypos.reshape(d, n)[:, first:first + count]
        assert np.array_equal(got.view(np.uint64), pos[:, first:first + count].view(np.uint64)), f"rank {rank}"
        assert passes < T + fails  # temporally blocked
