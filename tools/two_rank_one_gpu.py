"""Probe: two NCCL ranks on one GPU (two processes) driving sharded cuda-sync.
NCCL normally refuses duplicate GPUs; this checks what this image's NCCL does."""
import os, sys, json
import multiprocessing as mp
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, q, uid_q):
    import numpy as np
    import paper_2205_01313_b200 as cp
    f = cp.find_fitness("sphere")
    n, d, T = 20001, 8, 60
    p = cp.make_params(f, n, d, T)
    first, count = cp.shard_range(n, world, rank)
    try:
        sw = cp.Swarm(p, f, 5, device=0, first=first, count=count, init=False)
        if rank == 0:
            uid = cp.nccl_unique_id()
            for _ in range(world - 1):
                uid_q.put(uid)
        else:
            uid = uid_q.get(timeout=60)
        sw.nccl_init(uid, world, rank)
        sw.init()
        sw.step(cp.SYNC, 25)
        sw.step(cp.SYNC, T - 25)
        tr, tp, _ = sw.trace()
        q.put((rank, "ok", sw.sync_mode(), tr.tobytes().hex()[:64], int(tp[-1]), sw.spec_stats()))
    except Exception as e:
        q.put((rank, "error", repr(e)[:300], "", -1, None))


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ctx = mp.get_context("spawn")
    q, uq = ctx.Queue(), ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, q, uq)) for r in range(world)]
    for pr in ps:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in ps:
        pr.join(timeout=60)
    for r in sorted(res):
        print(r)
    import paper_2205_01313_b200 as cp
    f = cp.find_fitness("sphere")
    with cp.Swarm(cp.make_params(f, 20001, 8, 60), f, 5) as sw:
        sw.step(cp.SYNC, 60)
        tr, tp, _ = sw.trace()
        print("single", tr.tobytes().hex()[:64], int(tp[-1]))
