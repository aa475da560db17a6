#!/usr/bin/env python3
"""Benchmark of the per-gate decompress -> gate -> recompress hot path.

Headline workload (default, `--config C3`; BASELINE.json configs[2], SURVEY.md
§8d C3 -- the largest configuration that fits one GPU): QFT-34 on a seeded
basis state, 2^20-amplitude strides (16384 strides, 256 GiB uncompressed),
eps = 1e-3 mapped to the power-of-two absolute bound delta = 2^-27
(circuit.pow2_bound, <= SURVEY's eps*2^-17), single-level ladder, theta = 1.
The state at the start of the QFT's last stage (gate 612 of 646: qubits 0..32
transformed, qubit 33 still a basis bit -- the late, dense part of the
circuit) is built from its exact closed form (circuit.qft_stage) and
compressed by the engine (qcs_load_strides_device) -- untimed setup.  A *step*
is one gate of that last stage (CP(k, 33) ... H(33)), applied in circuit order
to the resident state; W warm-up steps, then K timed steps (wrapping to the
stage's first gate if W + K steps exceed its 34 gates).  The
state (>= 34 GB) is far larger than L2, so no flush is needed.

value     amplitude updates (sum of bytes_before/16, aalc.cpp:622) per second
          of DEVICE time (CUDA events on the engine's stream around every gate).
e2e       same metric through the public C-ABI call (qcs_run_program) from
          host gate descriptors to host GateRecords, host wall clock.
roofline  dominant kernel class, algorithmic bytes (C_in + C_out) / its
          event-timed duration vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline / same_shape
          the unmodified reference (oracle/_ref) on this host's cores at the
          same shape one size down (QFT-28, 2^20-amp strides, the same delta
          mapping, the same last-stage window, started from the same
          closed-form state compressed by the reference's own
          compress_stride_adaptive and CompressedState::load), and the GPU on
          exactly that state: both start from bit-identical amplitudes, so
          their GateRecords are compared field for field.

--impl reference runs the reference CPU path on that QFT-28 workload.
--config C2 is round 1's headline (Grover-24 gate form, 2^16-amp strides);
C1 / C3-full / C4s run a whole circuit once.  N > 1 (torchrun): the C2
workload weak-scaled to 24 + log2(N) qubits and sharded over the ranks.
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
from paper_1811_05140_b200.stage import load_stage_state, stage_fidelity  # noqa: E402

N_QUBITS, STRIDE_BITS, EPS, ITERS, SEED = 24, 16, 1e-4, 64, 7
GATES_PER_STEP = 2 * N_QUBITS + 2
RECORD_BYTES = 88
DESC_BYTES = 72
METRIC = "amplitude-updates/sec incl. codec (fused gate+codec HBM GB/s vs peak); fidelity; ratio"
UNIT = "amplitude-updates/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


EPS_MAPPING = "pow2"  # --eps-mapping (C2): "pow2" or "survey"


def c2_delta(n):
    return cc.survey_bound(EPS, n) if EPS_MAPPING == "survey" else cc.pow2_bound(EPS, n)


def workload(n=N_QUBITS):
    marked = next(cc.splitmix64(SEED)) & ((1 << n) - 1)
    prog = cc.build_grover_gate_form(n, marked, ITERS)
    delta = c2_delta(n)
    return prog, marked, delta


def config_dict(marked, delta, parallelism):
    return {
        "workload": "C2: grover-24 gate form, 64 iterations (3224 gates), 2^16-amp strides",
        "n_qubits": N_QUBITS, "stride_bits": STRIDE_BITS, "eps": EPS,
        "delta": delta, "delta_mapping": ("eps*2^-ceil(n/2) (SURVEY.md §8d)" if EPS_MAPPING == "survey"
                                          else "largest power of two <= eps*2^-ceil(n/2)"),
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


def measured_clock_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("sm_max_mhz", 1965.0))
    except (OSError, ValueError):
        return 1965.0


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
def dense_apply(psi, n, g):
    """One gate on a dense complex128 state (the uncompressed checker, after
    dense.cpp:30-76; torch complex arithmetic, so agreement is to rounding)."""
    import torch
    if g.kind == cc.KIND_FLIP:
        psi[g.flip_index] = -psi[g.flip_index]
        return
    if g.kind == cc.KIND_REFLECT:
        psi.copy_(2.0 * psi.mean() - psi)
        return
    u, t = g.unitary, g.target
    if g.kind == cc.KIND_SINGLE:
        v = psi.view(1 << (n - t - 1), 2, 1 << t)
        a0, a1 = v[:, 0, :].clone(), v[:, 1, :].clone()
        v[:, 0, :] = u.u11 * a0 + u.u12 * a1
        v[:, 1, :] = u.u21 * a0 + u.u22 * a1
        return
    c = g.control
    hi, lo = max(c, t), min(c, t)
    v = psi.view(1 << (n - hi - 1), 2, 1 << (hi - lo - 1), 2, 1 << lo)
    sel = (lambda b, x: v[:, 1, :, b, :]) if c == hi else (lambda b, x: v[:, b, :, 1, :])
    a0, a1 = sel(0, None).clone(), sel(1, None).clone()
    sel(0, None).copy_(u.u11 * a0 + u.u12 * a1)
    sel(1, None).copy_(u.u21 * a0 + u.u22 * a1)


def dense_state(prog, n_gates, device, basis=0):
    import torch
    n = prog.n_qubits
    psi = torch.zeros(1 << n, dtype=torch.complex128, device=device)
    psi[basis] = 1.0
    for g in prog.gates[:n_gates]:
        dense_apply(psi, n, g)
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


def cpu_baseline(prog, delta, first_iter):
    """Reference on this host's cores, on the GPU arm's own step: the H^24
    prologue and iterations 0..first_iter-1 untimed, then Grover iteration
    `first_iter` (50 gates) timed, workers = all cores."""
    ref, why = reference_lib()
    if ref is None:
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": why}
    text = cc.print_circuit(prog)
    st = ref.state(text, STRIDE_BITS, 0)
    a, b = step_range(first_iter)
    st.apply(0, a, [delta], 1.0, 0)
    r = st.apply(a, b, [delta], 1.0, 0)
    return {"value": r["amp_updates"] / (r["gate_ns"] * 1e-9), "unit": UNIT,
            "cores": ref.max_threads(), "kind": "reference",
            "sample": f"Grover iteration {first_iter} of C2 (gates {a}..{b - 1}) after the untimed prologue, "
                      f"{r['amp_updates']:.3e} amplitude updates in {r['gate_ns'] * 1e-9:.1f} s, "
                      "workers = all cores"}


def g_shift(n):
    """Fewer gates per step for larger states (each gate costs 2^n)."""
    return max(0, n - N_QUBITS)


def run_reference(args, rank, world):
    """The unmodified reference (oracle/_ref) on this host's cores, on the same
    workload as the B200 arm: C2, or at N > 1 the weak-scaled 24 + log2 N
    qubit state the sharded arm runs (rank 0 only)."""
    g = max(0, world.bit_length() - 1)
    n = N_QUBITS + g
    prog, marked, delta = workload(n)
    cfg = config_dict(marked, delta, "reference CPU, rank 0 only")
    if world > 1:
        cfg.update({"workload": f"C2 weak-scaled: grover-{n} gate form (the {world}-GPU arm's state)",
                    "n_qubits": n, "delta": delta, "ladder": [delta], "step": f"a window of the grover-{n} gates"})
    if rank != 0:
        return 0
    ref, why = reference_lib()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return 0
    text = cc.print_circuit(prog)
    st = ref.state(text, STRIDE_BITS, 0)
    st.apply(0, n, [delta], 1.0, 0)                            # untimed prologue
    gps = 2 * n + 2
    if n == N_QUBITS:
        # the GPU arm's steps: whole Grover iterations after the prologue
        steps = [(n + (i % ITERS) * gps, n + (i % ITERS + 1) * gps) for i in range(args.warmup + args.steps)]
        desc = f"{args.steps} Grover iterations ({gps} gates each) after the H^{n} prologue and {args.warmup} warm-up iterations"
    else:
        # weak-scaled state (N > 1 arms): bounded windows of consecutive gates
        total = args.warmup + args.steps
        g = gps if total <= 12 else max(10, (12 * gps) // total)
        g = max(4, g >> g_shift(n))
        steps, pos = [], n
        for _ in range(total):
            if pos + g > len(prog.gates):
                pos = n  # wrap (state keeps evolving; rate is what is measured)
            steps.append((pos, pos + g))
            pos += g
        desc = f"{args.steps} steps x {g} consecutive gates of grover-{n} after the H^{n} prologue"
    for a, b in steps[: args.warmup]:
        st.apply(a, b, [delta], 1.0, 0)
    ns = upd = 0.0
    wall0 = time.perf_counter()
    for a, b in steps[args.warmup:]:
        r = st.apply(a, b, [delta], 1.0, 0)
        ns += r["gate_ns"]
        upd += r["amp_updates"]
    wall = time.perf_counter() - wall0
    value = upd / (ns * 1e-9)
    cores = ref.max_threads()
    sample = f"{desc}, workers = {cores}"
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
def run_sharded(args, rank, world, local_rank):
    """N > 1: one state of 24 + log2(N) qubits sharded over the ranks (rank =
    top qubits), so per-GPU work equals the N = 1 workload
    (weak scaling).  Gates on rank qubits exchange stride images with NCCL
    send/recv (paper_1811_05140_b200/distributed.py); renormalisation and
    GateRecords are global.  Device time: CUDA events around the timed
    steps on every rank, max over ranks."""
    import torch
    import paper_1811_05140_b200 as q
    from paper_1811_05140_b200.distributed import GpuBackend, ShardedState, ShardGeometry, TorchComm

    g = world.bit_length() - 1
    if (1 << g) != world:
        raise SystemExit("--gpus must be a power of two")
    n = N_QUBITS + g
    marked = next(cc.splitmix64(SEED)) & ((1 << n) - 1)
    prog = cc.build_grover_gate_form(n, marked, ITERS)
    delta = c2_delta(n)
    gps = 2 * n + 2
    dev = 0 if os.environ.get("QCS_SAME_DEVICE") else local_rank
    torch.cuda.set_device(dev)
    comm = TorchComm()
    st = ShardedState(ShardGeometry(n, STRIDE_BITS, g), comm, GpuBackend(dev), 0)
    lad, th = [delta], 1.0
    for i in range(n):                                          # untimed prologue
        st.apply_gate(prog.gates[i], lad, th, i)

    def run_steps(first, count):
        upd = 0
        mr = math.inf
        for k in range(count):
            a = n + ((first + k) % ITERS) * gps
            for i in range(a, a + gps):
                rec, _ = st.apply_gate(prog.gates[i], lad, th, i)
                upd += rec.bytes_before // 16
                mr = min(mr, rec.min_ratio)
        return upd, mr

    run_steps(0, args.warmup)
    l0 = q.engine.lib().qcs_state_launches(st.local.h)
    torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                                 else ".", f"clocks_rank{rank}.csv"))
    if rank == 0:
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    upd, min_ratio = run_steps(args.warmup, args.steps)
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    wall = time.perf_counter() - w0
    torch.distributed.barrier()
    clk = clocks.stop() if rank == 0 else None
    launches = q.engine.lib().qcs_state_launches(st.local.h) - l0
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3, wall], dtype=torch.float64, device=torch.device("cuda", dev))
    if torch.distributed.get_backend() == "nccl":
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    else:
        tc = t.cpu()
        torch.distributed.all_reduce(tc, op=torch.distributed.ReduceOp.MAX)
        t = tc
    dev_s, wall_s = float(t[0]), float(t[1])
    if rank != 0:
        return 0
    peak, peak_src = measured_peaks()
    line = {"metric": METRIC, "value": upd / dev_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_s * 1e3 / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated circuit, seeded marked index)",
            "config": {"workload": f"C2 weak-scaled: grover-{n} gate form sharded over {world} GPUs "
                                   f"(2^{N_QUBITS} amplitudes per GPU, as at N=1)",
                       "n_qubits": n, "stride_bits": STRIDE_BITS, "eps": EPS, "delta": delta,
                       "delta_mapping": "largest power of two <= eps*2^-ceil(n/2)", "ladder": [delta],
                       "theta": 1.0, "marked": marked, "iterations": ITERS,
                       "step": f"one Grover iteration ({gps} gates)",
                       "l2": "per-GPU state 2^24 amplitudes; no explicit flush (exchange traffic between gates)",
                       "parallelism": f"{world} shards, rank = top {g} qubits, NCCL stride-image exchange"},
            "roofline": {"bound": "hbm", "achieved": None, "peak": peak, "unit": "GB/s", "frac": None,
                         "traffic": None, "peak_source": peak_src,
                         "note": "see the N=1 line for the kernel roofline"},
            "cpu_baseline": None,
            "e2e": {"value": upd / wall_s, "unit": UNIT, "h2d_bytes_per_step": DESC_BYTES * gps,
                    "d2h_bytes_per_step": 48 * (1 << (N_QUBITS - STRIDE_BITS)) * gps},
            "gpu_launches": launches, "clocks": clk, "min_stride_ratio": min_ratio}
    print(json.dumps(line))
    return 0


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
    # live event timing of the dominant kernel (the encoder) only: two events
    # per launch; events around every kernel cost ~5% of the step.  The other
    # classes' shares come from one untimed all-class pass after the run.
    state.profile(2)
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
    alg = {"decode": cin + raw, "serial_chain": raw + raw // 4, "fused": cin + cout, "commit": 2 * cout}
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

    # The encoder is issue/latency-bound, not HBM-bound: its
    # instruction roofline = profiled warp instructions per launch (ncu, same
    # command, profiles/) / the live event-timed launch time, against the issue
    # peak (148 SMs x 4 schedulers x max SM clock).
    ip = os.path.join(ROOT, "profiles", "r1_ncu_summary.json")
    if cls == "fused" and os.path.exists(ip):
        with open(ip) as f:
            prof = json.load(f)
        modes = [prof[k] for k in ("k_fused_local", "k_fused_raw") if k in prof]
        if modes:
            inst = sum(m["inst_executed"] for m in modes) / len(modes)
            peak_ips = 148 * 4 * measured_clock_mhz() * 1e6
            achieved_ips = inst / (t_cls / max(1, n_cls) * 1e-9)
            roofline["instruction_roofline"] = {
                "warp_inst_per_launch": inst, "achieved_warp_inst_per_s": achieved_ips,
                "peak_warp_inst_per_s": peak_ips, "frac": achieved_ips / peak_ips,
                "source": "inst_executed from profiles/r1_ncu_summary.json (mean of the two encoder modes); "
                          "peak = 148 SMs x 4 schedulers x sm_max_mhz"}

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
    # kernel shares of one more (untimed) iteration with every class timed
    it = (args.warmup + args.steps) % ITERS
    a, b = step_range(it)
    state.profile(1)
    q.apply_program_range(state, prog, a, b, lad, th)
    kt_all = state.kernel_times()
    state.profile(False)
    roofline["kernel_share"] = {k: v[0] / max(1.0, sum(x[0] for x in kt_all.values())) for k, v in kt_all.items()}
    roofline["kernel_share_source"] = "one untimed iteration after the timed run, events around every kernel"
    cpu = cpu_baseline(prog, delta, 1) if (world == 1 and not args.no_cpu_baseline) else None

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


# ---------------------------------------------------------------------------
# QFT configurations: the whole circuit once, fidelity
# against the closed-form DFT row a_y = exp(2 pi i (x*y mod 2^n)/2^n)/2^(n/2)
# (circuit.hpp:137-138), streamed from the device stride by stride.
# ---------------------------------------------------------------------------
QFT_CONFIGS = {
    "C1": dict(n=20, s=14, eps=1e-3, basis=552808, note="BASELINE configs[0]; basis = mt19937_64(1)() & (2^20-1)"),
    "C3": dict(n=34, s=20, eps=1e-3, basis=None, note="BASELINE configs[2]; 256 GiB uncompressed > one GPU"),
    # BASELINE configs[3] (6x6 = 36 qubits over 2-8 GPUs) at the largest grid one
    # B200 also holds uncompressed for the fidelity check: 5x6 = 30 qubits
    "C4s": dict(n=30, s=20, eps=1e-2, basis=0, grid=(5, 6, 20, 2024),
                note="BASELINE configs[3] shape (seeded NN-CZ + {sqrt X, sqrt Y, T} grid, depth 20) on 5x6 "
                     "qubits, one GPU; fidelity against a dense complex128 run on the same GPU"),
}


def qft_basis(name, n):
    c = QFT_CONFIGS[name]
    return c["basis"] if c["basis"] is not None else next(cc.splitmix64(n)) & ((1 << n) - 1)


def dense_fidelity(state, prog, n, s, x, device):
    """Fidelity |<dense|state>| / (|dense| |state|) against a dense complex128
    run of the same circuit on the GPU (dense.cpp:94-108), streamed stride by
    stride; also the largest amplitude difference."""
    import torch
    psi = dense_state(prog, len(prog.gates), device, basis=x)
    L, NS = 1 << s, 1 << (n - s)
    batch = max(1, min(NS, (1 << 28) // (16 * L)))
    buf = torch.empty(batch * 2 * L, dtype=torch.float64, device=device)
    ov = torch.zeros((), dtype=torch.complex128, device=device)
    nrm = torch.zeros((), dtype=torch.float64, device=device)
    maxerr = torch.zeros((), dtype=torch.float64, device=device)
    for j0 in range(0, NS, batch):
        m = min(batch, NS - j0)
        state.read_strides_device(j0, m, buf.data_ptr())
        v = buf[: m * 2 * L].view(m, 2, L)
        a = torch.complex(v[:, 0, :], v[:, 1, :]).reshape(-1)
        e = psi[j0 * L:(j0 + m) * L]
        ov += torch.sum(torch.conj(e) * a)
        nrm += torch.sum(a.real * a.real + a.imag * a.imag)
        maxerr = torch.maximum(maxerr, torch.max(torch.abs(a - e)))
    pn = torch.linalg.vector_norm(psi)
    del psi
    return float(torch.abs(ov) / (torch.sqrt(nrm) * pn)), float(maxerr)


def dft_fidelity(state, n, s, x, device):
    import torch
    L, NS = 1 << s, 1 << (n - s)
    batch = max(1, min(NS, (1 << 28) // (16 * L)))
    buf = torch.empty(batch * 2 * L, dtype=torch.float64, device=device)
    ov = torch.zeros((), dtype=torch.complex128, device=device)
    nrm = torch.zeros((), dtype=torch.float64, device=device)
    maxerr = torch.zeros((), dtype=torch.float64, device=device)
    mask = (1 << n) - 1
    xs = torch.tensor(x, dtype=torch.int64, device=device)
    inv = 1.0 / math.sqrt(float(1 << n))
    for j0 in range(0, NS, batch):
        m = min(batch, NS - j0)
        state.read_strides_device(j0, m, buf.data_ptr())
        v = buf[: m * 2 * L].view(m, 2, L)
        a = torch.complex(v[:, 0, :], v[:, 1, :])
        y = torch.arange(j0 * L, (j0 + m) * L, dtype=torch.int64, device=device).view(m, L)
        r = (xs * y) & mask                      # uint64 wrap-around product mod 2^n
        ph = r.to(torch.float64) * (2.0 * math.pi / float(1 << n))
        e = torch.complex(torch.cos(ph), torch.sin(ph)) * inv
        ov += torch.sum(torch.conj(e) * a)
        nrm += torch.sum(a.real * a.real + a.imag * a.imag)
        maxerr = torch.maximum(maxerr, torch.max(torch.abs(a - e)))
    # the reference's fidelity: |<a|b>| / (|a| |b|) (dense.cpp:94-108); |e| = 1
    return float(torch.abs(ov) / torch.sqrt(nrm)), float(maxerr)


def run_qft_config(args, name):
    import torch
    import paper_1811_05140_b200 as q
    c = QFT_CONFIGS[name]
    n, s = c["n"], c["s"]
    x = qft_basis(name, n)
    delta = cc.pow2_bound(c["eps"], n)
    prog = cc.build_grid(*c["grid"]) if "grid" in c else cc.build_qft(n)
    torch.cuda.set_device(0)
    lad = q.ErrorBoundLadder.make([delta])
    th = q.RatioThreshold(1.0)
    os.environ.setdefault("QCS_RESERVE_BYTES", str(8 << 30))  # room for the fidelity pass
    state = q.CompressedState.basis_state(q.StateGeometry.make(n, s), x)
    big = n > 24  # long kernels: the per-launch events cost nothing measurable, profile the timed run
    if big:
        state.profile(True)
    clocks = Clocks(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                                 else ".", f"clocks_{name}.csv"))
    clocks.start()
    dev_ns = upd = cin = cout = 0
    min_ratio = math.inf
    t0 = time.perf_counter()
    chunk = 16
    for a in range(0, len(prog.gates), chunk):
        m = q.apply_program_range(state, prog, a, min(len(prog.gates), a + chunk), lad, th)
        for r in m.records:
            dev_ns += r.elapsed_ns
            upd += r.bytes_before // 16
            cin += r.compressed_in
            cout += r.bytes_after
            min_ratio = min(min_ratio, r.min_ratio)
        if a % 128 == 0:
            log(f"{name}: {a + len(m.records)}/{len(prog.gates)} gates, {dev_ns * 1e-9:.1f} s device")
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    cbytes, min_stride, nsq = state._stats()
    if "grid" in c:
        fid, maxerr = dense_fidelity(state, prog, n, s, x, torch.device("cuda", 0))
    else:
        fid, maxerr = dft_fidelity(state, n, s, x, torch.device("cuda", 0))
    ctr = state.counters()
    # per-kernel-class device time (CUDA events around every launch): a second,
    # separate pass over the circuit so the events do not touch the timed one
    # (long configurations: the first gates only)
    if big:
        kt, n_prof = state.kernel_times(), len(prog.gates)
    else:
        prof = q.CompressedState.basis_state(q.StateGeometry.make(n, s), x)
        prof.profile(True)
        n_prof = len(prog.gates)
        q.apply_program_range(prof, prog, 0, n_prof, lad, th)
        kt = prof.kernel_times()
        del prof
    peak, peak_src = measured_peaks()
    # encoder time of one full pass over the circuit (the timed run for large
    # states, a separate profiled pass for small ones): C_in + C_out over it
    t_f, n_f = kt["fused"]
    t_f_run = t_f
    achieved = (cin + cout) / (t_f_run * 1e-9) / 1e9 if t_f_run else 0.0
    roofline = {"bound": "hbm", "kernel": "encoder (k_stream, k_fused)", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": (cin + cout) / max(1, n_f),
                "avg_launch_us": t_f_run / max(1, n_f) / 1e3,
                "launch_time_source": "CUDA events on the engine stream, " + (
                    "the timed run" if big else f"a second, profiled pass over the {n_prof} gates"),
                "kernel_share": {k: v[0] / max(1.0, sum(x_[0] for x_ in kt.values())) for k, v in kt.items()}}
    line = {"metric": METRIC, "value": upd / (dev_ns * 1e-9), "unit": UNIT, "n_gpus": 1,
            "steps": 1, "warmup": 0, "ms_per_step": dev_ns * 1e-6, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated " + ("seeded grid" if "grid" in c else "QFT") + " circuit, seeded basis state)",
            "config": {"workload": f"{name}: {prog.name} ({len(prog.gates)} gates), 2^{s}-amp strides",
                       "n_qubits": n, "stride_bits": s, "eps": c["eps"], "delta": delta,
                       "delta_mapping": "largest power of two <= eps*2^-ceil(n/2)", "basis": x,
                       "note": c["note"], "step": "the whole circuit once"},
            "e2e": {"value": upd / wall, "unit": UNIT, "h2d_bytes_per_step": DESC_BYTES * len(prog.gates),
                    "d2h_bytes_per_step": RECORD_BYTES * len(prog.gates)},
            ("fidelity_vs_dense" if "grid" in c else "fidelity_vs_dft_row"): fid,
            "max_abs_amp_error": maxerr, "pointwise_bound": delta,
            "norm_sq_tracked": nsq, "min_stride_ratio": min_ratio,
            "final_state_ratio": (16 << n) / cbytes, "final_compressed_bytes": cbytes,
            "bytes_per_amp_update": (cin + cout) / max(1, upd),
            "layout": {"wave_slots": ctr["wave_slots"], "compactions": ctr["compactions"],
                       "compaction_s": ctr["compaction_ns"] * 1e-9},
            "roofline": roofline, "codec_counters": {k: v for k, v in ctr.items() if k != "phase_cycles"},
            "gpu_launches": state.launches(), "clocks": clk}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# C3 headline: the last stage of QFT-34 on its exact intermediate state
# ---------------------------------------------------------------------------
# (a step is ONE gate of the last stage: the driver's --steps 20 --warmup 5 then stays inside the
# stage on both arms — 25 of its 34 gates at n = 34, 25 of 28 on the reference arm's n = 28 — with
# no wrap onto the state H(n-1) has made fully dense, and the fidelity check applies)
C3 = dict(n=34, s=20, eps=1e-3, ref_n=28, step=1, cpu_gates=12)


def c3_setup(n):
    """QFT-n, its seeded basis (round 1's C3 basis), the first gate of its last
    stage (CP(0, n-1) ... CP(n-2, n-1), H(n-1)) and the delta mapping."""
    prog = cc.build_qft(n)
    x = next(cc.splitmix64(n)) & ((1 << n) - 1)
    g0 = len(prog.gates) - n
    return prog, x, g0, cc.pow2_bound(C3["eps"], n)


def c3_step(n, g0, i):
    """Gate range of step i: C3['step'] consecutive gates of the last stage,
    wrapping to its first gate once the stage is used up."""
    per = n // C3["step"]
    a = g0 + (i % per) * C3["step"]
    return a, a + C3["step"]


def ref_csv_records(csv):
    """emit_csv rows -> (rows without elapsed_ns, sum elapsed_ns, amplitude updates)."""
    lines = csv.strip().splitlines()
    head = lines[0].split(",")
    ie, ib = head.index("elapsed_ns"), head.index("bytes_before")
    rows, ns, upd = [], 0, 0
    for ln in lines[1:]:
        f = ln.split(",")
        ns += int(f[ie])
        upd += int(f[ib]) // 16
        rows.append(",".join(f[:ie] + f[ie + 1:]))
    return rows, ns, upd


def same_shape_c3(q, ref, device, n_gates):
    """The reference (all host cores) and the GPU on the SAME QFT-28 state
    (2^20-amp strides, the same delta mapping): the closed-form state at the
    start of the last stage, compressed by each engine from bit-identical
    amplitudes, then the first n_gates gates of the stage.  Returns the CPU
    baseline, the GPU line and whether the GateRecords agree bit for bit."""
    from paper_1811_05140_b200 import metrics as mm
    import torch
    n, s = C3["ref_n"], C3["s"]
    prog, x, g0, delta = c3_setup(n)
    tables = cc.stage_tables(n, s, *cc.qft_stage(n, x, g0))
    path = os.path.join("/tmp", f"qcs_c3_ref{n}_{os.getpid()}.qckp")
    t0 = time.perf_counter()
    rst = ref.state_from_tables(cc.print_circuit(prog), s, tables, [delta], 1.0, path)
    build_s = time.perf_counter() - t0
    try:
        os.remove(path)
    except OSError:
        pass
    csv = rst.apply_csv(g0, g0 + n_gates, [delta], 1.0, 0)
    rows_ref, ns_ref, upd_ref = ref_csv_records(csv)
    cores = ref.max_threads()
    del rst
    lad, th = q.ErrorBoundLadder.make([delta]), q.RatioThreshold(1.0)
    gst = load_stage_state(q, n, s, x, g0, lad, th, device)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    m = q.apply_program_range(gst, prog, g0, g0 + n_gates, lad, th)
    wall = time.perf_counter() - w0
    rows_gpu = mm.emit_csv(m.records, with_elapsed=False).strip().splitlines()[1:]
    dev_ns = sum(r.elapsed_ns for r in m.records)
    upd = sum(r.bytes_before // 16 for r in m.records)
    del gst
    sample = (f"QFT-{n} (2^{s}-amp strides, delta {delta:g}), the first {n_gates} gates of its last stage "
              f"from the closed-form state at gate {g0} (compress_stride_adaptive + CompressedState::load, "
              f"{build_s:.1f} s untimed), workers = {cores}")
    cpu = {"value": upd_ref / (ns_ref * 1e-9), "unit": UNIT, "cores": cores, "kind": "reference",
           "sample": sample}
    gpu = {"value": upd / (dev_ns * 1e-9), "e2e": upd / wall, "unit": UNIT, "n_qubits": n,
           "gates": n_gates, "records_identical_to_reference": rows_gpu == rows_ref,
           "ratio_value_vs_reference": (upd / (dev_ns * 1e-9)) / (upd_ref / (ns_ref * 1e-9)),
           "ratio_e2e_vs_reference": (upd / wall) / (upd_ref / (ns_ref * 1e-9))}
    if rows_gpu != rows_ref:
        bad = next(i for i, (a, b) in enumerate(zip(rows_gpu, rows_ref)) if a != b) if len(rows_gpu) == len(rows_ref) else -1
        log("same-shape records differ at row", bad, rows_gpu[bad] if bad >= 0 else "", rows_ref[bad] if bad >= 0 else "")
    return cpu, gpu


def run_c3(args, rank, world, local_rank):
    import torch
    import paper_1811_05140_b200 as q
    n, s = C3["n"], C3["s"]
    prog, x, g0, delta = c3_setup(n)
    dev = local_rank
    torch.cuda.set_device(dev)
    os.environ.setdefault("QCS_RESERVE_BYTES", str(8 << 30))  # torch buffers of setup / fidelity
    lad, th = q.ErrorBoundLadder.make([delta]), q.RatioThreshold(1.0)
    t0 = time.perf_counter()
    state = load_stage_state(q, n, s, x, g0, lad, th, dev)
    setup_s = time.perf_counter() - t0
    log(f"C3 state at gate {g0} loaded in {setup_s:.1f} s: {state._stats()}")
    for i in range(args.warmup):
        a, b = c3_step(n, g0, i)
        q.apply_program_range(state, prog, a, b, lad, th)
    clocks = Clocks(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                                 else ".", f"clocks_rank{rank}.csv"))
    launches0 = state.launches()
    state.profile(2)          # events around the encoder launches only
    torch.cuda.synchronize()
    clocks.start()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ (launch lists)
    dev_ns = wall_ns = 0
    upd = cin = cout = 0
    min_ratio = math.inf
    last_gate = g0
    for i in range(args.warmup, args.warmup + args.steps):
        a, b = c3_step(n, g0, i)
        torch.cuda.synchronize()
        w0 = time.perf_counter_ns()
        m = q.apply_program_range(state, prog, a, b, lad, th)   # C-ABI: host descs in, records out
        wall_ns += time.perf_counter_ns() - w0
        for r in m.records:
            dev_ns += r.elapsed_ns
            upd += r.bytes_before // 16
            cin += r.compressed_in
            cout += r.bytes_after
            min_ratio = min(min_ratio, r.min_ratio)
        last_gate = b
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    clk = clocks.stop()
    kt = state.kernel_times()
    log("kernel times (ns, launches):", kt)
    state.profile(False)
    launches = state.launches() - launches0
    wrapped = (args.warmup + args.steps) * C3["step"] > n
    fid = maxerr = None
    if not args.skip_fidelity and not wrapped:
        fid, maxerr = stage_fidelity(state, n, s, x, last_gate, dev)
    cbytes, min_stride, nsq = state._stats()
    arena, side_b, scratch_b = state.memory()
    ctr = state.counters()
    # kernel shares of one more (untimed) step with every class timed
    state.profile(1)
    a, b = c3_step(n, g0, args.warmup + args.steps)
    q.apply_program_range(state, prog, a, b, lad, th)
    kt_all = state.kernel_times()
    state.profile(False)
    del state
    torch.cuda.empty_cache()

    peak, peak_src = measured_peaks()
    t_f, n_f = kt["fused"]
    achieved = (cin + cout) / (t_f * 1e-9) / 1e9 if t_f else 0.0
    path_gbs = (cin + cout) / (dev_ns * 1e-9) / 1e9
    traffic = None
    streamed = ctr.get("stream_slots", 0) > 0
    tp = os.path.join(ROOT, "profiles", "traffic_k_stream_c3.json" if streamed else "traffic_k_fused_c3.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        # DRAM bytes per algorithmic byte of the captured launch (ncu --set full),
        # applied to this run's algorithmic bytes per launch
        if tj.get("traffic_per_algorithmic_byte"):
            traffic = tj["traffic_per_algorithmic_byte"] * (cin + cout) / max(1, n_f)
    tot_all = max(1.0, sum(v[0] for v in kt_all.values()))
    # (wave layout, single-level ladder: the persistent form of the streaming kernel)
    roofline = {"bound": "hbm", "kernel": ("k_stream_persist" if ctr["wave_slots"] else "k_stream") if streamed else "k_fused",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": (f"ncu --set full of the encoder on the C3 shape at n = 28 (tools/profile_c3.py, "
                                   f"profiles/{os.path.basename(tp)}): its DRAM bytes per algorithmic byte "
                                   "times this run's algorithmic bytes per launch") if traffic else None,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": (cin + cout) / max(1, n_f),
                "algorithmic_bytes": "C_in + C_out of the gates' rewritten strides, 29-byte headers included "
                                     "(SURVEY.md §8d), over the encoder launches of the timed steps (per gate one "
                                     "persistent launch of the streaming kernel, then per wave the legacy encoder k_fused "
                                     "for the slots it left, timed together)",
                "encoder_slots": {"streamed": ctr.get("stream_slots", 0),
                                  "left_to_legacy_encoder": ctr.get("stream_left_slots", 0)},
                "avg_launch_us": t_f / max(1, n_f) / 1e3,
                "path_C_in_plus_C_out_GBps": path_gbs, "path_frac": path_gbs / peak,
                "kernel_share": {k: v[0] / tot_all for k, v in kt_all.items()},
                "kernel_share_source": "one untimed step after the timed run, events around every kernel"}
    cpu = same = None
    if world == 1 and not args.no_cpu_baseline:
        ref, why = reference_lib()
        if ref is None:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": why}
        else:
            cpu, same = same_shape_c3(q, ref, dev, C3["cpu_gates"])
    line = {"metric": METRIC, "value": upd / (dev_ns * 1e-9), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ns * 1e-6 / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference-built QFT circuit, seeded basis, exact closed-form stage state)",
            "config": {"workload": f"C3: qft-{n}, last stage (gates {g0}..{len(prog.gates) - 1}) on the "
                                   f"exact state at gate {g0}, 2^{s}-amp strides, one B200",
                       "n_qubits": n, "stride_bits": s, "eps": C3["eps"], "delta": delta,
                       "delta_mapping": "largest power of two <= eps*2^-ceil(n/2) (SURVEY.md: eps*2^-17)",
                       "ladder": [delta], "theta": 1.0, "basis": x,
                       "step": ("one gate" if C3["step"] == 1 else f"{C3['step']} consecutive gates") + " of the last stage",
                       "wrapped": wrapped,
                       "l2": "state (>= 34 GB) larger than L2; no flush", "parallelism": "single GPU",
                       "setup": f"closed-form state compressed on the GPU ({setup_s:.1f} s, untimed)"},
            "roofline": roofline, "cpu_baseline": cpu, "same_shape": same,
            "e2e": {"value": upd / (wall_ns * 1e-9), "unit": UNIT,
                    "h2d_bytes_per_step": DESC_BYTES * C3["step"],
                    "d2h_bytes_per_step": RECORD_BYTES * C3["step"]},
            "gpu_launches": launches, "clocks": clk,
            "fidelity_vs_exact": fid, "max_abs_amp_error": maxerr, "pointwise_bound": delta,
            "min_stride_ratio": min_ratio, "final_state_ratio": (16 << n) / cbytes,
            "compressed_bytes": cbytes, "hbm_bytes": {"arena_in_use": arena, "side_index": side_b,
                                                      "scratch": scratch_b},
            "layout": {"wave_slots": ctr["wave_slots"], "compactions": ctr["compactions"],
                       "compaction_s": ctr["compaction_ns"] * 1e-9},
            "bytes_per_amp_update": (cin + cout) / max(1, upd)}
    print(json.dumps(line))
    return 0


def run_reference_c3(args, rank, world):
    """The unmodified reference on this host's cores at the same shape one size
    down (QFT-28, 2^20-amp strides, the delta mapping of n = 28): the closed-form
    state at the start of the last stage, compressed by the reference's own
    compress_stride_adaptive and read by CompressedState::load, then steps of 2
    consecutive last-stage gates through apply_program_range (rank 0 only)."""
    if rank != 0:
        return 0
    ref, why = reference_lib()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return 0
    n, s = C3["ref_n"], C3["s"]
    prog, x, g0, delta = c3_setup(n)
    path = os.path.join("/tmp", f"qcs_c3_ref{n}_{os.getpid()}.qckp")
    t0 = time.perf_counter()
    st = ref.state_from_tables(cc.print_circuit(prog), s, cc.stage_tables(n, s, *cc.qft_stage(n, x, g0)),
                               [delta], 1.0, path)
    build_s = time.perf_counter() - t0
    try:
        os.remove(path)
    except OSError:
        pass
    for i in range(args.warmup):
        a, b = c3_step(n, g0, i)
        st.apply(a, b, [delta], 1.0, 0)
    ns = upd = 0.0
    wall0 = time.perf_counter()
    for i in range(args.warmup, args.warmup + args.steps):
        a, b = c3_step(n, g0, i)
        r = st.apply(a, b, [delta], 1.0, 0)
        ns += r["gate_ns"]
        upd += r["amp_updates"]
    wall = time.perf_counter() - wall0
    value = upd / (ns * 1e-9)
    cores = ref.max_threads()
    sample = (f"QFT-{n} (2^{s}-amp strides, delta {delta:g}), {args.steps} steps x {C3['step']} gates of the "
              f"last stage from the closed-form state at gate {g0} (compress_stride_adaptive + "
              f"CompressedState::load, {build_s:.1f} s untimed), workers = {cores}")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ns * 1e-6 / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference-built QFT circuit, seeded basis, exact closed-form stage state)",
            "config": {"workload": f"C3 shape one size down: qft-{n} last stage, 2^{s}-amp strides "
                                   "(the B200 arm's C3 workload at n = 34 costs the same per amplitude; "
                                   "SURVEY.md §8d same-shape method)",
                       "n_qubits": n, "stride_bits": s, "eps": C3["eps"], "delta": delta,
                       "delta_mapping": "largest power of two <= eps*2^-ceil(n/2)", "ladder": [delta],
                       "theta": 1.0, "basis": x,
                       "step": ("one gate" if C3["step"] == 1 else f"{C3['step']} consecutive gates") + " of the last stage",
                       "parallelism": "reference CPU (OpenMP), rank 0 only"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": upd / wall, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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
    ap.add_argument("--config", default="C3", choices=["C3", "C2", "C1", "C3-full", "C4s"],
                    help="C3 (default): the headline, QFT-34's last stage on one GPU; C2: Grover-24 gate "
                         "form; C1 / C3-full: a whole QFT once; C4s: the 30-qubit grid")
    ap.add_argument("--eps-mapping", default="pow2", choices=["pow2", "survey"],
                    help="C2 only: delta = largest power of two <= eps*2^-ceil(n/2) (default) or "
                         "SURVEY.md's eps*2^-ceil(n/2) itself")
    args = ap.parse_args()
    global EPS_MAPPING
    EPS_MAPPING = args.eps_mapping
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config in ("C1", "C3-full", "C4s"):
        return run_qft_config(args, "C3" if args.config == "C3-full" else args.config)
    if args.config == "C3" and world == 1:
        if args.impl == "reference":
            return run_reference_c3(args, rank, world)
        return run_c3(args, rank, world, local_rank)
    if args.warmup < 3 and args.impl == "b200":
        log("warning: timing rules ask for >= 3 warm-up steps")
    if world > 1:
        import torch
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("QCS_DIST_BACKEND", "nccl" if args.impl == "b200" else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group(backend)
    try:
        if args.impl == "reference":
            return run_reference(args, rank, world)
        if world > 1:
            return run_sharded(args, rank, world, local_rank)
        return run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
