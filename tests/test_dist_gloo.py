"""World-size-2 multi-process test of the sharded path's host logic on CPU
(gloo).  Each rank plans the circuit with libqs's planner (qs_plan_json; the
plan must be identical on every rank, as rank mode requires), keeps only its
own shard, and performs every global<->local swap as a real all-to-all over
the process group with the same piece routing as exec_swap (piece s of rank r
goes to rank r with the swapped bits := s, landing at piece u(r)).  The
gathered result must equal the oracle."""
import math
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import json
        import paper_2604_12256_b200 as qs
        import workloads as W
        from tests import plan_replay as PR

        gates = W.qaoa_maxcut(n, 2, seed) + W.random_circuit(n, 60, seed, diag_bias=0.3)
        plan = qs.plan_json(n, gates, n_ranks=world, product_state=True, basis=3, detail=True)
        # every rank must hold the same plan
        blob = json.dumps(plan, sort_keys=True)
        allp = [None] * world
        dist.all_gather_object(allp, blob)
        assert all(p == blob for p in allp)
        g = int(math.log2(world))
        nl = n - g
        # Run the plan with single-rank replay for everything but swaps: we
        # split the plan at swap steps and exchange shards over gloo.
        shard = None
        steps = plan["steps"]
        seg = []
        state = {"shards": None}

        subs = {}

        def run_segment(seg_steps, shards_in):
            sub = dict(plan)
            sub["steps"] = seg_steps
            return PR.replay_shards(sub, n, world, shards_in, subs)

        for st in steps + [{"type": "end"}]:
            if st["type"] in ("swap", "end"):
                shards = run_segment(seg, state["shards"])
                seg = []
                mine = shards[rank]
                if st["type"] == "swap":
                    j = st["j"]
                    bits = [p - nl for p in st["gpos"]]
                    piece = 1 << (nl - j)
                    ur = sum(((rank >> b) & 1) << i for i, b in enumerate(bits))
                    send = [torch.zeros(2 * piece, dtype=torch.float64) for _ in range(world)]
                    recv = [torch.zeros(2 * piece, dtype=torch.float64) for _ in range(world)]
                    for s in range(1 << j):
                        d = rank
                        for i, b in enumerate(bits):
                            d = (d & ~(1 << b)) | (((s >> i) & 1) << b)
                        send[d] = torch.from_numpy(mine[s * piece:(s + 1) * piece].view(np.float64).copy())
                    # grouped point-to-point exchange, as exec_swap does with
                    # ncclSend/ncclRecv (gloo has no all_to_all)
                    reqs = []
                    for d in range(world):
                        if d == rank:
                            recv[d] = send[d].clone()
                        else:
                            reqs.append(dist.isend(send[d], d))
                            reqs.append(dist.irecv(recv[d], d))
                    for rq in reqs:
                        rq.wait()
                    new = np.empty_like(mine)
                    for src in range(world):
                        # partners agree on the non-swapped rank bits; rank src
                        # sent us its piece u(rank), which lands at piece u(src)
                        same = all((src >> k) & 1 == (rank >> k) & 1
                                   for k in range(g) if k not in bits)
                        if same:
                            us = sum(((src >> b) & 1) << i for i, b in enumerate(bits))
                            new[us * piece:(us + 1) * piece] = recv[src].numpy().view(np.complex128)
                    mine = new
                # only our shard is authoritative; others are placeholders
                state["shards"] = [mine if r == rank else np.zeros_like(mine) for r in range(world)]
            else:
                seg.append(st)
        full = [torch.zeros(2 << nl, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(full, torch.from_numpy(state["shards"][rank].view(np.float64).copy()))
        if rank == 0:
            shards = [t.numpy().view(np.complex128) for t in full]
            mp_ = plan["map_out"]
            L = np.arange(1 << n, dtype=np.int64)
            phys = np.zeros_like(L)
            for qq in range(n):
                phys |= ((L >> qq) & 1) << mp_[qq]
            psi = np.concatenate(shards)[phys]
            import oracle
            want = oracle.apply_circuit(n, gates, x=3)
            q.put(float(np.max(np.abs(psi - want))))
    except Exception as e:  # surface errors to the parent
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,seed", [(8, 1), (12, 2)])
def test_gloo_world2_sharded_plan(n, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + n
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(res, str), res
    assert res < 1e-11
