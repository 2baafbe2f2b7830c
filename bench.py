"""bench.py -- driver benchmark of the state-vector hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload qft|rzz|diag|qaoa|rand] [--no-cpu-baseline]

One "step" = one pass of the whole hot path over one synthetic input:
qs_set_basis_state(x) + qs_apply_circuit(circuit) through the C-ABI
(host optimiser: booster, diagonal detector, blocking, fusion; then the
device passes / swaps).  Workload (BASELINE.json configs[1]): the n-qubit QFT
(reading c18) from |x>, n = 30 + log2(N) (weak scaling: a 16 GiB shard per
GPU).  Inputs (the gate list, marshalled once) are resident before the timed
region; the state (16 GiB per GPU) is far larger than the 126 MB L2, so no L2
flush is needed between steps.

Printed value: effective HBM GB/s of the whole job = sum over GPUs of the
plan's algorithmic bytes (32 B per amplitude per read+write pass, 16 B per
write-only pass) / device time per step.  ms_per_step is the
circuit wall time measured with CUDA events on the library's launching stream
(max over ranks).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "circuit wall time and effective HBM GB/s at 30–35 qubits, 1/2/4/8 B200"
BASIS_X = 0x2A5F3C71


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(workload: str, kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of this workload's dominant kernel from the committed ncu --set full
    capture (profiles/traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        e = d[workload][kernel]
        return e["bytes_per_launch"]
    except Exception:
        return None


def make_circuit(workload: str, n: int):
    import workloads as W
    if workload == "qft":
        return W.qft(n)
    if workload == "rzz":
        return W.rzz_full(n, 1)
    if workload == "diag":
        return W.diag_chain(n, 1)
    if workload == "qaoa":
        return W.qaoa_maxcut(n, 4, 1, degree=3 if n % 2 == 0 else 4)
    if workload == "rand":  # BASELINE configs[4]: supremacy-style, depth 20 (5x7 grid at 35)
        return W.supremacy(5, 7, 20, 1) if n == 35 else W.supremacy_n(n, 20, 1)
    raise ValueError(workload)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region of a short workload can be ~50 ms: wait until
            # the sampler is producing before it starts
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Start of the timed region: only samples from here on count."""
        self.n0 = len(self.lines)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        n0 = getattr(self, "n0", 0)
        # samples of the timed region; a region shorter than the 20 ms
        # sampling interval keeps the sample just before it
        for ln in (self.lines[n0:] if len(self.lines) > n0 else self.lines[max(0, n0 - 1):]):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# Algorithmic HBM bytes (whole job) of this build's plan for each bench
# config: the byte count both arms divide by, so the driver's value ratio is
# the circuit-time ratio.  A constant here (checked against the planner by
# tests/test_bench_contract.py) so the reference arm never loads libqs.
PLAN_BYTES = {
    "qft30": 51539607552, "qft31": 103079215104, "qft32": 206158430208, "qft33": 412316860416,
    "rzz30": 17179869184, "rzz31": 34359738368, "rzz32": 68719476736, "rzz33": 137438953472,
    "diag30": 51539607552, "diag31": 103079215104, "diag32": 206158430208, "diag33": 412316860416,
    "qaoa30": 360777252864, "qaoa31": 858993459200, "qaoa32": 1855425871872, "qaoa33": 3710851743744,
    "rand30": 1288490188800, "rand31": 2783138807808, "rand32": 5841155522560, "rand33": 12781822672896,
}


def host_info() -> dict:
    model, mem_kb = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                mem_kb = int(ln.split()[1])
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gib": round(mem_kb / 2 ** 20, 1) if mem_kb else None,
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS")}


class OracleSampler:
    """The oracle as it stands (gate-by-gate Alg. 1) on the
    FULL state of the bench config, timed on a bounded, evenly strided
    sample of the circuit's gates; the circuit time is the sample time
    scaled by G / |sample| (each gate is one sweep of the whole state, and
    the oracle's time per gate does not depend on the amplitude values)."""

    def __init__(self, workload: str, n: int):
        import numpy as np
        import oracle
        oracle.build()
        self.oracle = oracle
        self.n_circuit = n
        self.G = len(make_circuit(workload, n))
        # a state that does not fit in ~45% of the available host memory (e.g.
        # 33 qubits = 128 GiB) is sampled on the largest one that does; each
        # gate is one sweep of the state, so the circuit time scales by
        # 2^(n - n_eff) * G(n) / G(n_eff)
        avail = None
        try:
            for ln in open("/proc/meminfo"):
                if ln.startswith("MemAvailable"):
                    avail = int(ln.split()[1]) * 1024
        except OSError:
            pass
        self.n = n
        while avail is not None and (16 << self.n) > 0.45 * avail and self.n > 20:
            self.n -= 1
        self.gates = make_circuit(workload, self.n)
        self.scale = (2.0 ** (n - self.n)) * self.G / len(self.gates)
        self.psi = oracle.basis_state(self.n, BASIS_X % (1 << self.n))
        # first touch of every page + the per-gate time estimate (untimed)
        oracle.apply_circuit(self.n, self.gates[:1], state=self.psi, inplace=True)
        t0 = time.perf_counter()
        oracle.apply_circuit(self.n, self.gates[1:2], state=self.psi, inplace=True)
        self.t_gate = max(1e-4, time.perf_counter() - t0)
        self.np = np

    def sample(self, budget_s: float) -> dict:
        G = len(self.gates)
        k = int(max(2, min(G, budget_s / self.t_gate)))
        stride = max(1, G // k)
        sub = self.gates[::stride]
        t0 = time.perf_counter()
        self.oracle.apply_circuit(self.n, sub, state=self.psi, inplace=True)
        dt = time.perf_counter() - t0
        return {"circuit_s": dt * G / len(sub) * self.scale, "sample_s": dt, "sample_gates": len(sub),
                "stride": stride, "gates": G, "n_state": self.n}


def cpu_baseline(workload: str, n: int, budget_s: float = 15.0) -> dict:
    """cpu_baseline of the JSON line: the oracle on the bench config (all
    host cores), plus a single-thread leg at n = 26."""
    import oracle
    key = "%s%d" % (workload, n)
    oracle.set_num_threads(os.cpu_count() or 1)
    s = OracleSampler(workload, n)
    r = s.sample(budget_s)
    del s
    out = {"value": PLAN_BYTES[key] / r["circuit_s"] / 1e9, "unit": "GB/s", "cores": oracle.num_threads(),
           "kind": "oracle",
           "sample": "%s (%d gates, full 2^%d state): every %d-th gate (%d gates) applied by the oracle in "
                     "%.1f s on %d threads; circuit time %.1f s = sample x G/|sample|; value = this build's plan "
                     "bytes for %s (%.4g GB, bench.PLAN_BYTES) / circuit time"
                     % (key, r["gates"], n, r["stride"], r["sample_gates"], r["sample_s"], oracle.num_threads(),
                        r["circuit_s"], key, PLAN_BYTES[key] / 1e9),
           "circuit_s": r["circuit_s"], "host": host_info()}
    # single-threaded leg at n = 26 (the same workload), a few seconds
    n1 = min(n, 26)
    oracle.set_num_threads(1)
    try:
        s1 = OracleSampler(workload, n1)
        r1 = s1.sample(min(6.0, budget_s / 2))
        del s1
    finally:
        oracle.set_num_threads(out["cores"])
    out["single_thread"] = {"workload": "%s%d" % (workload, n1), "circuit_s": r1["circuit_s"],
                            "sample_gates": r1["sample_gates"], "gates": r1["gates"]}
    return out


def run_reference(args):
    """--impl reference: the CPU oracle (the tier's reference arm) on the GPU
    arm's config; each step is a bounded strided gate sample of that
    circuit on the full state (OracleSampler), scaled to the circuit; rank 0
    only.  Never loads libqs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    g = int(round(math.log2(max(1, world))))
    n = args.n or (30 + g)
    key = "%s%d" % (args.workload, n)
    per_step = max(2.0, min(15.0, 150.0 / max(1, args.steps + args.warmup)))
    # torchrun exports OMP_NUM_THREADS=1: the reference arm runs on all the
    # host's cores, like the N = 1 leg
    oracle.set_num_threads(os.cpu_count() or 1)
    s = OracleSampler(args.workload, n)
    for _ in range(args.warmup):
        s.sample(per_step)
    times = [s.sample(per_step) for _ in range(args.steps)]
    circ = sum(t["circuit_s"] for t in times) / len(times)
    val = PLAN_BYTES[key] / circ / 1e9
    sample = ("%s: per step every %d-th gate (%d of %d) of the %d-qubit circuit on its full 2^%d state, %.1f s, "
              "scaled by G/|sample|%s; value = this build's plan bytes for %s / the scaled circuit time"
              % (key, times[0]["stride"], times[0]["sample_gates"], times[0]["gates"], s.n, s.n,
                 times[0]["sample_s"],
                 "" if s.n == n else " x 2^%d x G(%d)/G(%d) (host RAM: the %d-qubit state does not fit)"
                 % (n - s.n, n, s.n, n), key))
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": circ * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": key, "n_qubits": n, "gates": len(s.gates),
                   "note": "CPU oracle (gate-by-gate Alg. 1) on the GPU arm's workload; circuit time "
                           "extrapolated from a strided gate sample per step"},
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="qft", choices=["qft", "rzz", "diag", "qaoa", "rand"])
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=0,
                    help="override qubit count (--qubits under torchrun: its parser claims --n)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    import paper_2604_12256_b200 as qs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = int(round(math.log2(world)))
    n = args.n or (30 + g)
    gates = make_circuit(args.workload, n)
    marsh = qs.marshal_gates(gates)
    x = BASIS_X % (1 << n)

    # cold start (PAPER.md L382 bounds the optimiser at < 1/1000 of the run):
    # the first call with an EMPTY kernel cache compiles every specialised
    # pass (NVRTC, in parallel); later calls reuse the loaded kernels
    if not os.environ.get("QS_JIT_CACHE"):
        import tempfile
        os.environ["QS_JIT_CACHE"] = tempfile.mkdtemp(prefix="qs_jit_cold_")
    if world > 1:
        obj = [qs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        sim = qs.Simulator(n, rank=rank, world_size=world, device=local, nccl_id=obj[0])
    else:
        sim = qs.Simulator(n, device=local)
    stream = torch.cuda.ExternalStream(sim.stream(0), device=torch.device("cuda", local))

    def step():
        sim.set_basis_state(x)
        sim.apply(gates, marshalled=marsh)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    t_cold = time.perf_counter()
    step()
    torch.cuda.synchronize()
    cold_ms = (time.perf_counter() - t_cold) * 1e3
    jit0 = qs.jit_info(sim)
    for _ in range(max(3, args.warmup) - 1):
        step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # the library accumulates launches, per-kernel timings and plan/device
    # times over the timed steps (qs_set_timing(ctx, 2)): the loop holds
    # nothing but the steps, the totals are read once afterwards
    sim.set_timing(2)
    clocks.mark()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    barrier()
    launches = sim.launches()
    st_acc = sim.stats()
    plan_ms = st_acc["t_plan_ms"]
    dev_ms = st_acc["t_device_ms"]
    kt = {}
    for k in ("K1_chunk", "K2_dense", "K3_diag", "small", "K5_expand", "K5_merge", "init", "K4_swap",
              "substate", "fused_swap_pass", "pull_pass", "l2_group"):
        kt[k] = sim.kernel_timing(k)
    sim.set_timing(1)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = sim.stats()
    ms_t = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    bytes_per_step = st["bytes_hbm"] * world
    value = bytes_per_step / (ms * 1e-3) / 1e9

    # global<->local exchanges (K4): NVLink bytes each GPU sends per step;
    # fused swaps ride on the preceding pass's stores (their time is inside
    # that pass), so only unfused swaps have an exchange time of their own
    nvl = None
    if world > 1 and st["n_swaps"]:
        sw = kt.get("K4_swap", {"ms": 0.0, "launches": 0})
        fp = dict(kt.get("fused_swap_pass", {"ms": 0.0, "launches": 0, "bytes": 0}))
        pp = kt.get("pull_pass", {"ms": 0.0, "launches": 0, "bytes": 0})
        # a split swap's exchange is spread over the exporting pass and the
        # pass after it (push/pull): both carry NVLink traffic
        fp = {k2: fp.get(k2, 0) + pp.get(k2, 0) for k2 in ("ms", "launches", "bytes")}
        unf = st["n_swaps"] - st["n_fused_swaps"]
        per_swap = st["bytes_nvlink"] / st["n_swaps"]   # (1 - 2^-j) x shard bytes per swap (equal j here)
        nvl = {"bytes_per_gpu_per_step": st["bytes_nvlink"], "swaps": st["n_swaps"],
               "fused_swaps": st["n_fused_swaps"], "swap_step_ms": sw["ms"] / args.steps,
               "peak_gbs_per_direction": 900.0,
               "peak_source": "NVLink 5 spec, per direction per GPU (PAPER.md L709 quotes 900 GB/s NVSwitch "
                              "for the DGX-H100; no measured NVLink peak on file)"}
        if st["n_fused_swaps"] and fp["ms"] > 0:
            # the fused pass moves its exported pieces over NVLink while it
            # streams the shard through HBM: the transfer time is at most the
            # pass time, so bytes / pass time is a LOWER bound of its NVLink rate
            b = per_swap * st["n_fused_swaps"]
            t = fp["ms"] / args.steps * 1e-3
            nvl["fused"] = {"nvlink_bytes_per_step": b, "pass_ms_per_step": t * 1e3,
                            "achieved_gbs_lower_bound": b / t / 1e9, "frac_of_900": b / t / 1e9 / 900.0,
                            "hbm_gbs_of_the_passes": fp["bytes"] / args.steps / t / 1e9}
        if unf and sw["ms"] > 0 and unf == st["n_swaps"]:
            nvl["nccl"] = {"achieved_gbs": st["bytes_nvlink"] / (sw["ms"] / args.steps * 1e-3) / 1e9}

    # dominant kernel (largest device time) -> roofline
    dom = max(kt.items(), key=lambda kv: kv[1]["ms"])
    peak, peak_src = measured_peaks()
    roof = None
    if dom[1]["launches"]:
        avg_ms = dom[1]["ms"] / dom[1]["launches"]
        per_launch = dom[1]["bytes"] / dom[1]["launches"]
        ach = per_launch / (avg_ms * 1e-3) / 1e9
        if dom[0] == "K4_swap":
            roof = {"kernel": dom[0], "bound": "nvlink", "achieved": ach, "peak": 900.0,
                    "peak_source": "NVLink 5 spec, per direction per GPU (no measured NVLink peak on file)",
                    "unit": "GB/s", "frac": ach / 900.0, "traffic": None}
        else:
            roof = {"kernel": dom[0], "bound": "hbm", "achieved": ach, "peak": peak,
                    "peak_source": peak_src + " (MEASURED_PEAKS.json hbm_gbs, burst copy)",
                    "unit": "GB/s", "frac": ach / peak, "traffic": measured_traffic(
                        "%s%d" % (args.workload, n), dom[0]),
                    "bytes_per_launch": per_launch, "avg_launch_ms": avg_ms,
                    "share_of_step": dom[1]["ms"] / args.steps / ms}

    # e2e: through the C-ABI with host buffers: gate list marshalled from the
    # Python objects every step (host), descriptors H2D, a 1 Mi-amplitude
    # slice of the result state D2H (host buffer).
    e2e = None
    if args.e2e_steps > 0:
        slice_amps = 1 << 20
        # the result slice lands in pinned host memory (DMA, no staging copy)
        host_out = torch.empty(slice_amps, dtype=torch.complex128, pin_memory=True).numpy()
        # untimed warm-up of the readout path (NCCL all-reduce setup in rank mode)
        sim.set_basis_state(x)
        sim.apply(gates, marshalled=marsh)
        sim.state(0, slice_amps, out=host_out)
        barrier()
        t0 = time.perf_counter()
        h2d = 0
        for _ in range(args.e2e_steps):
            sim.set_basis_state(x)
            m2 = qs.marshal_gates(gates)
            h2d += 104 * len(gates)  # qs_gate_t records consumed by the library
            sim.apply(gates, marshalled=m2)
            out = sim.state(0, slice_amps, out=host_out)
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        t_e = torch.tensor([e2e_ms], device="cuda")
        if dist is not None:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e_ms = float(t_e.item())
        e2e = {"value": bytes_per_step / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d // args.e2e_steps,
               "d2h_bytes_per_step": slice_amps * 16,
               "note": "set_basis_state + marshal + qs_apply_circuit + qs_get_state(1 Mi amps)"}

    if rank == 0:
        base = None
        if not args.no_cpu_baseline and world == 1:
            base = cpu_baseline(args.workload, n)
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s%d" % (args.workload, n), "n_qubits": n, "gates": len(gates),
                       "basis": x, "shard_gib": (16 << (n - g)) / 2 ** 30,
                       "parallelism": "state sharded by top %d qubits over %d GPU(s)" % (g, world),
                       "l2": "no flush: state %.0f GiB per GPU >> 126 MB L2" % ((16 << (n - g)) / 2 ** 30)},
            "circuit_ms": ms, "device_busy_ms_per_step": dev_ms / args.steps,
            "plan_ms_per_step": plan_ms / args.steps,
            "plan": {k: st[k] for k in ("n_passes", "n_chunk_passes", "n_dense_passes",
                                        "n_diag_passes", "n_swaps", "n_expand",
                                        "n_substate_gates", "n_fused_diag", "bytes_hbm")},
            "kernels": {k: v for k, v in kt.items() if v["launches"]},
            "roofline": roof, "cpu_baseline": base, "e2e": e2e, "nvlink": nvl,
            "gpu_launches": launches, "clocks": clk,
            "cold_start": {"first_call_ms": cold_ms, "compile_ms": jit0["compile_ms"],
                           "compiles": jit0["compiles"], "prep_ms": jit0["prep_ms"],
                           "host_threads": os.cpu_count(),
                           "note": "first qs_apply_circuit with an empty kernel cache (NVRTC compiles of "
                                   "every pass structure, parallel over host threads; compile_ms sums the "
                                   "per-kernel compile times) vs circuit_ms once compiled"},
            "jit_variants": qs.jit_info(sim)["variants"],
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
