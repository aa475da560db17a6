#!/usr/bin/env python3
"""Benchmark of the per-gate decompress -> gate -> recompress hot path.

Workload (BASELINE.json configs[1]): 24-qubit Grover search in
gate form, H^24 then 64 x [flip m; H^24; flip 0; H^24] (3224 gates),
2^16-amplitude strides, error bound eps = 1e-4 mapped to the power-of-two
absolute bound delta = 2^-26 (circuit.pow2_bound), single-level ladder,
theta = 1, marked index m seeded (SplitMix64, seed 7).  Synthetic: the
circuit is generated, no external data.

A *step* is one Grover iteration (50 gates) applied to the resident state;
the H^24 prologue is untimed setup.  W warm-up steps, then K timed steps;
the state keeps evolving along the circuit.  L2 is flushed (256 MiB write)
before every timed step.

value     amplitude updates (sum of bytes_before/16, aalc.cpp:622) per second
          of DEVICE time (CUDA events on the engine's stream around every gate),
          state resident in HBM.
e2e       same metric through the public C-ABI call (qcs_run_program) from
          host gate descriptors to host GateRecords, host wall clock.
roofline  dominant kernel class, algorithmic bytes / its event-timed duration
          vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the unmodified reference (oracle/_ref/libqcsref.so) on this
          host's cores, bounded sample of the same circuit.

--impl reference runs the reference CPU path on the same workload instead.
N > 1 (torchrun): independent replicas, one per GPU (the C2 state fits one
GPU; the sharded multi-GPU path is DESIGN.md §7), max device time over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1811_05140_b200 import circuit as cc  # noqa: E402

N_QUBITS, STRIDE_BITS, EPS, ITERS, SEED = 24, 16, 1e-4, 64, 7
GATES_PER_STEP = 2 * N_QUBITS + 2
RECORD_BYTES = 88
DESC_BYTES = 72
METRIC = "amplitude-updates/sec incl. codec (fused gate+codec HBM GB/s vs peak); fidelity; ratio"
UNIT = "amplitude-updates/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload():
    marked = next(cc.splitmix64(SEED)) & ((1 << N_QUBITS) - 1)
    prog = cc.build_grover_gate_form(N_QUBITS, marked, ITERS)
    delta = cc.pow2_bound(EPS, N_QUBITS)
    return prog, marked, delta


def config_dict(marked, delta, parallelism):
    return {
        "workload": "C2: grover-24 gate form, 64 iterations (3224 gates), 2^16-amp strides",
        "n_qubits": N_QUBITS, "stride_bits": STRIDE_BITS, "eps": EPS,
        "delta": delta, "delta_mapping": "largest power of two <= eps*2^-ceil(n/2)",
        "ladder": [delta], "theta": 1.0, "marked": marked, "iterations": ITERS,
        "step": f"one Grover iteration ({GATES_PER_STEP} gates)",
        "l2": "flushed before each timed step (256 MiB write)",
        "parallelism": parallelism,
    }


def step_range(i):
    a = N_QUBITS + i * GATES_PER_STEP
    return a, a + GATES_PER_STEP


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, out_path):
        self.path = out_path
        self.p = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# dense checker for fidelity (torch on the GPU; test-side only)
# ---------------------------------------------------------------------------
def dense_state(prog, n_gates, device):
    import torch
    n = prog.n_qubits
    psi = torch.zeros(1 << n, dtype=torch.complex128, device=device)
    psi[0] = 1.0
    for g in prog.gates[:n_gates]:
        if g.kind == cc.KIND_FLIP:
            psi[g.flip_index] = -psi[g.flip_index]
        elif g.kind == cc.KIND_SINGLE:
            u = g.unitary
            v = psi.view(1 << (n - g.target - 1), 2, 1 << g.target)
            a0, a1 = v[:, 0, :].clone(), v[:, 1, :].clone()
            v[:, 0, :] = u.u11 * a0 + u.u12 * a1
            v[:, 1, :] = u.u21 * a0 + u.u22 * a1
        else:
            raise NotImplementedError("bench dense checker covers the C2 gate set")
    return psi


# ---------------------------------------------------------------------------
# CPU legs (the unmodified reference, compiled by oracle/Makefile)
# ---------------------------------------------------------------------------
def reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Reference
    if not Reference.available():
        return None, "oracle/_ref/libqcsref.so not built (needs /root/reference at build time)"
    return Reference(), None


def cpu_baseline(prog, delta):
    """Reference on this host's cores: H^24 prologue + the first iteration
    (74 gates) of the same circuit, workers = all cores."""
    ref, why = reference_lib()
    if ref is None:
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": why}
    text = cc.print_circuit(prog)
    st = ref.state(text, STRIDE_BITS, 0)
    last = N_QUBITS + GATES_PER_STEP
    r = st.apply(0, last, [delta], 1.0, 0)
    return {"value": r["amp_updates"] / (r["gate_ns"] * 1e-9), "unit": UNIT,
            "cores": ref.max_threads(), "kind": "reference",
            "sample": f"gates 0..{last} of C2 (H^24 prologue + 1 iteration), "
                      f"{r['amp_updates']:.3e} amplitude updates in {r['gate_ns'] * 1e-9:.1f} s, "
                      "workers = all cores"}


def run_reference(args, rank, world):
    prog, marked, delta = workload()
    cfg = config_dict(marked, delta, "reference CPU, rank 0 only")
    if rank != 0:
        return 0
    ref, why = reference_lib()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return 0
    text = cc.print_circuit(prog)
    st = ref.state(text, STRIDE_BITS, 0)
    st.apply(0, N_QUBITS, [delta], 1.0, 0)                     # untimed prologue
    total = args.warmup + args.steps
    g = GATES_PER_STEP if total <= 12 else max(10, (12 * GATES_PER_STEP) // total)
    pos = N_QUBITS
    for _ in range(args.warmup):
        st.apply(pos, pos + g, [delta], 1.0, 0)
        pos += g
    ns = upd = 0.0
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        if pos + g > len(prog.gates):
            pos = N_QUBITS  # wrap (state keeps evolving; rate is what is measured)
        r = st.apply(pos, pos + g, [delta], 1.0, 0)
        pos += g
        ns += r["gate_ns"]
        upd += r["amp_updates"]
    wall = time.perf_counter() - wall0
    value = upd / (ns * 1e-9)
    cores = ref.max_threads()
    sample = f"{args.steps} steps x {g} consecutive C2 gates after the H^24 prologue, workers = {cores}"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ns * 1e-6 / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated circuit, seeded marked index)", "config": cfg,
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": upd / wall, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args, rank, world, local_rank):
    import torch
    import paper_1811_05140_b200 as q
    from paper_1811_05140_b200.engine import lib

    prog, marked, delta = workload()
    dev = local_rank
    torch.cuda.set_device(dev)
    geom = q.StateGeometry.make(N_QUBITS, STRIDE_BITS)
    lad = q.ErrorBoundLadder.make([delta])
    th = q.RatioThreshold(1.0)
    state = q.CompressedState.basis_state(geom, 0, device=dev)
    q.apply_program_range(state, prog, 0, N_QUBITS, lad, th)   # untimed prologue
    for i in range(args.warmup):
        a, b = step_range(i % ITERS)
        q.apply_program_range(state, prog, a, b, lad, th)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                                 else ".", f"clocks_rank{rank}.csv"))
    launches0 = state.launches()
    state.profile(True)
    barrier()
    if rank == 0:
        clocks.start()
    dev_ns = wall_ns = 0.0
    upd = cin = cout = 0
    min_ratio = math.inf
    for i in range(args.steps):
        it = (args.warmup + i) % ITERS
        a, b = step_range(it)
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter_ns()
        m = q.apply_program_range(state, prog, a, b, lad, th)     # C-ABI: host descs in, records out
        wall_ns += time.perf_counter_ns() - t0
        for r in m.records:
            dev_ns += r.elapsed_ns
            upd += r.bytes_before // 16
            cin += r.compressed_in
            cout += r.bytes_after
            min_ratio = min(min_ratio, r.min_ratio)
    barrier()
    clk = clocks.stop() if rank == 0 else None
    kt = state.kernel_times()
    log("kernel times (ns, launches):", kt)
    log("codec counters:", state.counters())
    state.profile(False)
    launches = state.launches() - launches0

    # max over ranks of device time; sum of work
    if world > 1:
        t = torch.tensor([dev_ns, wall_ns], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_max, wall_max = float(t[0]), float(t[1])
        w = torch.tensor([float(upd)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(w)
        upd_all = float(w[0])
    else:
        dev_max, wall_max, upd_all = dev_ns, wall_ns, float(upd)
    if rank != 0:
        return 0

    value = upd_all / (dev_max * 1e-9)
    e2e = upd_all / (wall_max * 1e-9)
    peak, peak_src = measured_peaks()
    # dominant kernel class
    cls, (t_cls, n_cls) = max(kt.items(), key=lambda kv: kv[1][0])
    L = 1 << STRIDE_BITS
    raw = upd * 16                                # uncompressed bytes of rewritten strides
    # k_fused reads the compressed input strides and writes the recompressed ones
    # (algorithmic bytes = C_in + C_out); commit copies C_out
    alg = {"decode": cin + raw, "gate": 2 * raw, "fused": cin + cout, "commit": 2 * cout}
    alg_bytes = alg.get(cls, cin + cout)
    achieved = alg_bytes / (t_cls * 1e-9) / 1e9 if t_cls else 0.0
    path_gbs = (cin + cout) / (dev_ns * 1e-9) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_k_{cls}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f)["traffic_bytes"]
    roofline = {"bound": "hbm", "kernel": f"k_{cls}", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_source": "ncu --set full, one launch (profiles/)" if traffic else None,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes / max(1, n_cls),
                "avg_launch_us": t_cls / max(1, n_cls) / 1e3,
                "path_C_in_plus_C_out_GBps": path_gbs, "path_frac": path_gbs / peak,
                "kernel_share": {k: v[0] / max(1.0, sum(x[0] for x in kt.values())) for k, v in kt.items()}}

    fidelity = None
    if not args.skip_fidelity:
        n_applied = N_QUBITS + (args.warmup + args.steps) * GATES_PER_STEP
        if args.warmup + args.steps <= ITERS:
            import numpy as np
            psi = dense_state(prog, n_applied, dev)
            amps = torch.from_numpy(state.to_amplitudes()).to(dev)
            fidelity = float(torch.abs(torch.vdot(psi, amps)) / (torch.linalg.vector_norm(psi) *
                                                                 torch.linalg.vector_norm(amps)))
            del psi, amps
    cbytes, min_stride, _ = state._stats()
    cpu = cpu_baseline(prog, delta) if (world == 1 and not args.no_cpu_baseline) else None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_max * 1e-6 / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated circuit, seeded marked index)",
            "config": config_dict(marked, delta, "single GPU" if world == 1 else f"{world} replicas"),
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": UNIT,
                    "h2d_bytes_per_step": DESC_BYTES * GATES_PER_STEP,
                    "d2h_bytes_per_step": RECORD_BYTES * GATES_PER_STEP},
            "gpu_launches": launches, "clocks": clk,
            "fidelity": fidelity, "min_stride_ratio": min_ratio,
            "final_state_ratio": (16 << N_QUBITS) / cbytes,
            "bytes_per_amp_update": (cin + cout) / max(1, upd)}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-fidelity", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        log("warning: timing rules ask for >= 3 warm-up steps")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if args.impl == "b200" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group(backend)
    try:
        if args.impl == "reference":
            return run_reference(args, rank, world)
        return run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
