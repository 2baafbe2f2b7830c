"""Multi-GPU parity check (run under torchrun, one process per GPU).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/mgpu_check.py

Rank mode (qs_create_rank + NCCL swaps) on random, QAOA and QFT circuits vs
the CPU oracle on rank 0 (every rank receives the logical state through
qs_get_state, which is collective).  Rank 0 also checks the single-process
multi-device mode (qs_create(n, world)) when it can see every GPU.
Prints one JSON line per case; exits non-zero on a mismatch.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    import oracle
    import paper_2604_12256_b200 as qs
    import workloads as W

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def new_id():
        # every NCCL communicator needs its own unique id
        obj = [qs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    cases = [
        ("random18", 18, W.random_circuit(18, 250, 3, diag_bias=0.3)),
        ("qaoa20", 20, W.qaoa_maxcut(20, 3, 2)),
        ("qft21", 21, W.qft(21)),
        ("supremacy20", 20, W.supremacy(4, 5, 8, 1)),
        ("random22", 22, W.random_circuit(22, 300, 4, diag_bias=0.4)),
    ]
    bad = 0
    for name, n, gates in cases:
        for jit in (99, 0):
            cfg = qs.make_config(jit_min_qubits=jit)
            sim = qs.Simulator(n, rank=rank, world_size=world, device=local, nccl_id=new_id(), config=cfg)
            sim.set_basis_state(5)
            sim.apply(gates)
            psi = sim.state()
            st = sim.stats()
            sim.close()
            if rank == 0:
                want = oracle.apply_circuit(n, gates, x=5)
                err = float(np.max(np.abs(psi - want)))
                ok = err < 1e-12
                bad += not ok
                print(json.dumps({"case": name, "n": n, "world": world, "jit_min": jit, "max_abs_diff": err,
                                  "swaps": st["n_swaps"], "fused_swaps": st["n_fused_swaps"], "passes": st["n_passes"], "ok": ok}), flush=True)
    # large: QFT closed form at 28 + log2(world) qubits, sampled
    n = 28 + int(math.log2(world))
    x = 123456789 % (1 << n)
    sim = qs.Simulator(n, rank=rank, world_size=world, device=local, nccl_id=new_id())
    sim.set_basis_state(x)
    sim.apply(W.qft(n))
    st = sim.stats()
    worst = 0.0
    for off in (0, (1 << n) // 3, (1 << n) - 8192):
        got = sim.state(off, 8192)
        k = np.arange(off, off + 8192, dtype=np.int64)
        want = np.exp(2j * math.pi * ((x * k) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        worst = max(worst, float(np.max(np.abs(got - want))))
    sim.close()
    if rank == 0:
        ok = worst < 1e-12
        bad += not ok
        print(json.dumps({"case": "qft%d_closed_form" % n, "world": world, "max_abs_diff": worst,
                          "swaps": st["n_swaps"], "fused_swaps": st["n_fused_swaps"], "passes": st["n_passes"], "t_swap_ms": st["t_swap_ms"],
                          "t_device_ms": st["t_device_ms"], "ok": ok}), flush=True)
    # forced swaps: a circuit that touches the global qubits with dense gates
    n = 24
    gates = []
    for layer in range(4):
        gates += [W.Gate("RX", (q,), (), (0.1 + 0.01 * q + layer,)) for q in range(n)]
        gates += [W.Gate("CZ", (q + 1,), (q,)) for q in range(n - 1)]
    sim = qs.Simulator(n, rank=rank, world_size=world, device=local, nccl_id=new_id())
    sim.apply(gates)
    psi = sim.state()
    st = sim.stats()
    sim.close()
    if rank == 0:
        want = oracle.apply_circuit(n, gates)
        err = float(np.max(np.abs(psi - want)))
        ok = err < 1e-12 and (world == 1 or st["n_swaps"] >= 1)
        bad += not ok
        print(json.dumps({"case": "rx_layers24", "world": world, "max_abs_diff": err, "swaps": st["n_swaps"], "fused_swaps": st["n_fused_swaps"],
                          "bytes_nvlink": st["bytes_nvlink"], "t_swap_ms": st["t_swap_ms"], "ok": ok}),
              flush=True)
    # steady state at scale: QAOA and supremacy-style circuits on 26 qubits
    # (>= 22 local qubits: specialised kernels, many chunks per CTA, fused
    # swaps over NVLink peer stores), default configuration, vs the oracle
    for name, n, gates in (("qaoa26", 26, W.qaoa_maxcut(26, 3, 26)),
                           ("supremacy26", 26, W.supremacy_n(26, 8, 26))):
        sim = qs.Simulator(n, rank=rank, world_size=world, device=local, nccl_id=new_id())
        sim.apply(gates)
        psi = sim.state()
        st = sim.stats()
        sim.close()
        if rank == 0:
            err = float(np.max(np.abs(psi - oracle.apply_circuit(n, gates))))
            ok = err < 1e-12 and (world == 1 or st["n_swaps"] >= 1)
            bad += not ok
            print(json.dumps({"case": name, "world": world, "max_abs_diff": err, "swaps": st["n_swaps"],
                              "fused_swaps": st["n_fused_swaps"], "passes": st["n_passes"], "ok": ok}), flush=True)
    dist.barrier()
    if rank == 0 and torch.cuda.device_count() >= world:
        # single-process multi-device mode (ncclCommInitAll)
        n = 20
        gates = W.qaoa_maxcut(n, 3, 9)
        sim = qs.Simulator(n, n_gpus=world)
        sim.apply(gates)
        psi = sim.state()
        st = sim.stats()
        sim.close()
        err = float(np.max(np.abs(psi - oracle.apply_circuit(n, gates))))
        ok = err < 1e-12
        bad += not ok
        print(json.dumps({"case": "single_process_%dgpu" % world, "max_abs_diff": err,
                          "swaps": st["n_swaps"], "fused_swaps": st["n_fused_swaps"], "ok": ok}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
