"""Sharded state across ranks.

Rank = the top g = log2(world) qubits of the amplitude index, i.e. the top g
bits of the stride index: rank r holds global strides [r*NSL, (r+1)*NSL) as an
ordinary local engine state of n-g qubits with the same stride bits.  The
reference has no distribution; this layer reproduces its
single-process semantics exactly:

* gates on local qubits run unchanged on every rank; a control on a rank
  qubit turns into "this rank applies the uncontrolled gate or nothing",
  which is what make_stride_plan's control-bit skip does (gate.cpp:351-379);
* a target on a rank qubit b: partner ranks r and r^(1<<b) swap rank bit b
  with a local stride bit (half of each rank's strides change hands as
  device stride images: blocks verbatim with side index, scale and sum), and
  the ordinary cross-stride pair unit runs locally (aalc.cpp:333-382); the
  qubit permutation stays (no swap back; Belady eviction over the program);
* the lazy renormalisation (aalc.cpp:410-419) is global: per-stride
  (scale, sum_sq) are all-gathered and summed serially in global stride
  order, so every world size reproduces the single-GPU bits;
* GateRecords fold the stride reports in the reference's global unit order
  (aalc.cpp:612-631).

Exchanges move device stride images (qcs_pack_strides_range /
qcs_unpack_strides) point to point: NCCL send/recv over NVLink under
torch.distributed, staged through host memory on gloo.  The per-gate folds
(renormalisation, mean, records) are a host round trip here; the C++ driver
in the library (qcs_cluster_*, csrc/qcs_cluster.cuh) does them on the device
from one process.  The local engine is pluggable: GpuBackend (this package) or
the oracle's backend in oracle/oracle.py (CPU tests with gloo).
"""
from __future__ import annotations

import math
import os
import pickle
import struct
import threading
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .circuit import KIND_CONTROLLED, KIND_FLIP, KIND_REFLECT, KIND_SINGLE, GateOp
from .metrics import GateRecord


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class ThreadGroup:
    """Shared state for ranks running as threads of one process."""

    def __init__(self, size: int):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots: List[object] = [None] * size
        self.p2p = {}


class ThreadComm:
    def __init__(self, group: ThreadGroup, rank: int):
        self.group, self.rank, self.size = group, rank, group.size

    def allgather(self, obj):
        g = self.group
        g.slots[self.rank] = obj
        g.barrier.wait()
        out = list(g.slots)
        g.barrier.wait()
        return out

    def allgather_array(self, arr: np.ndarray) -> List[np.ndarray]:
        return self.allgather(np.array(arr, copy=True))

    def exchange(self, peer: Optional[int], obj, device: bool = False):
        """Collective: every rank calls it; peer None = no partner."""
        g = self.group
        if peer is not None:
            g.p2p[(self.rank, peer)] = obj
        g.barrier.wait()
        got = g.p2p.pop((peer, self.rank)) if peer is not None else None
        g.barrier.wait()
        return got


class TorchComm:
    """torch.distributed (gloo) communicator for host-staged exchanges."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allgather(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def allgather_array(self, arr: np.ndarray) -> List[np.ndarray]:
        """Equal-shape float64 arrays, through device tensors on NCCL."""
        import torch
        dev = (torch.device("cuda", torch.cuda.current_device())
               if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu"))
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(dev)
        out = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def exchange(self, peer: Optional[int], obj, device: bool = False):
        """Pairwise exchange.  device=True: device tensors (stride images) go
        point to point between the pair only (NCCL send/recv over NVLink;
        staged through host memory on gloo) and ranks without a partner do
        nothing.  Otherwise objects go through an all-gather every rank joins."""
        import torch
        if device:
            if peer is None:
                return None
        else:
            got = self.allgather((peer, obj))
            if peer is None:
                return None
            p_peer, p_obj = got[peer]
            assert p_peer == self.rank, "asymmetric exchange"
            return p_obj
        dist = self.dist
        nccl = dist.get_backend(self.group) == "nccl"
        dev = obj.device if nccl else torch.device("cpu")
        send = obj if nccl else obj.cpu()
        n_send = torch.tensor([send.numel()], dtype=torch.int64, device=dev)
        n_recv = torch.empty_like(n_send)
        self._p2p(send=n_send, recv=n_recv, peer=peer)
        recv = torch.empty(int(n_recv.item()), dtype=torch.uint8, device=dev)
        self._p2p(send=send, recv=recv, peer=peer)
        if nccl:
            # the engine reads the image on its own stream: wait on the host
            # until the receive (ordered on torch's stream by wait()) landed
            torch.cuda.current_stream().synchronize()
        return recv if nccl else recv.to(obj.device)

    def _p2p(self, send, recv, peer):
        dist = self.dist
        gp = peer if self.group is None else dist.get_global_rank(self.group, peer)
        ops = [dist.P2POp(dist.isend, send, gp, self.group), dist.P2POp(dist.irecv, recv, gp, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()


# ---------------------------------------------------------------------------
# local engine backends
# ---------------------------------------------------------------------------
class GpuBackend:
    """Local shard on a GPU through the C-ABI."""

    def __init__(self, device: int = 0):
        self.device = device

    def create(self, n: int, s: int, basis: Optional[int]):
        import ctypes as C
        from .engine import _check, lib
        h = C.c_void_p()
        b = (1 << 64) - 1 if basis is None else basis
        _check(lib().qcs_state_create(n, s, C.c_uint64(b), self.device, C.byref(h)))
        return _GpuShard(h, n, s, self.device)


# qcs_stride_report (include/qcs_b200.h) as a numpy record
_REPORT_DTYPE = np.dtype([("stride", "<u8"), ("b_in", "<u8"), ("b_out", "<u8"), ("delta", "<f8"),
                          ("ratio", "<f8"), ("met", "<i4"), ("pad", "<i4")])


class _GpuShard:
    device_images = True  # stride images are device tensors (point-to-point exchange)

    def __init__(self, h, n, s, device=0):
        self.h, self.n, self.s, self.device = h, n, s, device

    def __del__(self):
        try:
            from .engine import _lib_handle
        except Exception:  # interpreter shutdown: modules already torn down
            return
        if getattr(self, "h", None) and _lib_handle is not None:
            _lib_handle.qcs_state_destroy(self.h)
            self.h = None

    def apply(self, gate: GateOp, ladder, theta, mean=None):
        import ctypes as C
        from .circuit import pack_gates
        from .engine import Report, _check, lib
        reps = (Report * (1 << (self.n - self.s)))()
        nr = C.c_uint64()
        norm = C.c_double()
        lad = (C.c_double * len(ladder))(*ladder)
        m = (C.c_double * 2)(*(mean or (0.0, 0.0)))
        flags = 1 | (2 if mean else 0)   # QCS_NO_RENORM | QCS_GIVEN_MEAN
        _check(lib().qcs_apply_gate_ex(self.h, pack_gates([gate]), lad, len(ladder), theta, flags,
                                       m, reps, C.byref(nr), C.byref(norm)))
        a = np.frombuffer(reps, dtype=_REPORT_DTYPE, count=nr.value)
        return np.stack([a["stride"].astype(np.float64), a["delta"], a["ratio"], a["b_in"].astype(np.float64),
                         a["b_out"].astype(np.float64), (a["met"] != 0).astype(np.float64)], axis=1)

    def stride_sums(self):
        from .engine import _check, lib
        p = np.empty(2 << (self.n - self.s))
        _check(lib().qcs_stride_sums(self.h, p.ctypes.data))
        return p

    def stride_norms(self):
        from .engine import _check, lib
        L = lib()
        ns = 1 << (self.n - self.s)
        sc = np.empty(ns)
        sm = np.empty(ns)
        _check(L.qcs_stride_norms(self.h, sc.ctypes.data, sm.ctypes.data))
        return sc, sm

    def scale_all(self, f: float):
        from .engine import _check, lib
        _check(lib().qcs_scale_all(self.h, f))

    def export(self, j: int):
        import ctypes as C
        from .engine import _check, lib
        n, sc, ss = C.c_uint64(), C.c_double(), C.c_double()
        _check(lib().qcs_export_blocks(self.h, j, None, 0, C.byref(n), C.byref(sc), C.byref(ss)))
        buf = C.create_string_buffer(n.value)
        _check(lib().qcs_export_blocks(self.h, j, buf, n.value, C.byref(n), C.byref(sc),
                                       C.byref(ss)))
        return buf.raw[: n.value], sc.value, ss.value

    def import_(self, j: int, blob: bytes, scale: float, ssq: float):
        from .engine import _check, lib
        _check(lib().qcs_import_blocks(self.h, j, blob, len(blob), scale, ssq))

    def pack(self, bit: int, value: int, first: int = 0, count: int = (1 << 64) - 1):
        """Device image of the strides with stride bit `bit` == value (those at
        positions [first, first + count) among them)."""
        import ctypes as C
        import torch
        from .engine import _check, lib
        n = C.c_uint64()
        _check(lib().qcs_pack_strides_range(self.h, bit, value, first, count, None, 0, C.byref(n)))
        t = torch.empty(n.value, dtype=torch.uint8, device=torch.device("cuda", self.device))
        _check(lib().qcs_pack_strides_range(self.h, bit, value, first, count, t.data_ptr(), n.value, C.byref(n)))
        return t

    def image_bytes(self, bit: int, value: int) -> int:
        import ctypes as C
        from .engine import _check, lib
        n = C.c_uint64()
        _check(lib().qcs_pack_strides(self.h, bit, value, None, 0, C.byref(n)))
        return n.value

    def unpack(self, img, xor_mask: int):
        from .engine import _check, lib
        _check(lib().qcs_unpack_strides(self.h, img.data_ptr(), img.numel(), xor_mask))

    def amplitudes(self):
        from .engine import _check, lib
        a = np.empty(2 << self.n, dtype=np.float64)
        _check(lib().qcs_to_amplitudes(self.h, a.ctypes.data))
        return a.view(np.complex128)


# ---------------------------------------------------------------------------
# the sharded state
# ---------------------------------------------------------------------------
@dataclass
class ShardGeometry:
    n_qubits: int
    stride_bits: int
    rank_bits: int

    @property
    def local_qubits(self) -> int:
        return self.n_qubits - self.rank_bits

    @property
    def local_strides(self) -> int:
        return 1 << (self.local_qubits - self.stride_bits)


class ShardedState:
    """Lazy qubit permutation over the stride bits: logical stride bit p lives
    at physical position pi[p]; positions [0, Q-s) are a rank's local stride
    bits, [Q-s, n-s) the rank bits.  A gate whose target sits on a rank bit
    swaps it with a local stride bit (one exchange, least recently used local
    qubit evicted) and the permutation stays — no swap back, so a rank-qubit
    gate costs one exchange.  In-stride qubits never move.  Records, the
    renormalisation and reflect_mean's mean are folded in LOGICAL global stride
    order, amplitudes() returns the logical state."""

    def __init__(self, geom: ShardGeometry, comm, backend, basis: int):
        if (1 << geom.rank_bits) != comm.size:
            raise ValueError("world size must be 2^rank_bits")
        if geom.local_qubits < geom.stride_bits + 1:
            raise ValueError("each rank needs at least two strides")
        self.geom, self.comm, self.r = geom, comm, comm.rank
        Q = geom.local_qubits
        mine = (basis >> Q) == self.r
        self.local = backend.create(Q, geom.stride_bits, basis & ((1 << Q) - 1) if mine else None)
        self.norm_sq = 1.0
        nb = geom.n_qubits - geom.stride_bits       # stride-index bits
        self.pi = list(range(nb))                   # logical -> physical
        self.inv = list(range(nb))                  # physical -> logical
        self.last_use = [-1] * nb                   # logical bit -> last gate index
        self.exchanges = 0
        self.next_target = None                     # schedule: per logical bit, sorted gate indices
        # exchange images are streamed in chunks of at most this many bytes
        self.exchange_chunk_bytes = int(os.environ.get("QCS_EXCHANGE_CHUNK_BYTES", str(2 << 30)))

    def set_schedule(self, gates) -> None:
        """Future target uses of every stride qubit, so an eviction can drop the
        local qubit needed furthest in the future (Belady) instead of the least
        recently used one."""
        s = self.geom.stride_bits
        nt = [[] for _ in self.pi]
        for i, g in enumerate(gates):
            if g.kind in (KIND_SINGLE, KIND_CONTROLLED) and g.target >= s:
                nt[g.target - s].append(i)
        self.next_target = nt

    def _next_use(self, p: int, index: int) -> int:
        import bisect
        uses = self.next_target[p]
        k = bisect.bisect_right(uses, index)
        return uses[k] if k < len(uses) else 1 << 62

    # -- index maps -----------------------------------------------------------
    def _phys_to_log(self, jp: np.ndarray) -> np.ndarray:
        return self._p2l_table()[jp]

    def _p2l_table(self) -> np.ndarray:
        """Physical -> logical global stride index for every stride, cached
        until the permutation changes (exchanges are rare)."""
        key = tuple(self.pi)
        if getattr(self, "_p2l_key", None) != key:
            jp = np.arange(1 << len(self.pi), dtype=np.int64)
            jl = np.zeros_like(jp)
            for p, q in enumerate(self.pi):
                jl |= ((jp >> q) & 1) << p
            self._p2l, self._p2l_key = jl, key
            self._log_order = np.argsort(jl)  # physical indices in logical order
        return self._p2l

    def _logical_order(self) -> np.ndarray:
        self._p2l_table()
        return self._log_order

    def _log_to_phys(self, j: int) -> int:
        out = 0
        for p, q in enumerate(self.pi):
            out |= ((j >> p) & 1) << q
        return out

    # -- data movement: swap rank bit b with local stride bit qb ------------
    def _swap(self, b: int, qb: int):
        """All ranks (the layout is global).  The lo rank of each pair sends its
        strides with local bit qb = 1, the hi rank those with qb = 0; each lands
        at j ^ 2^qb on the other side.  Streamed in chunks of strides (the same
        chunking on every rank: the smallest choice) so the images stay
        below exchange_chunk_bytes: received chunk c overwrites exactly the
        positions sent in chunk c."""
        r = self.r
        peer = r ^ (1 << b)
        send_bit = 0 if (r >> b) & 1 else 1
        device = getattr(self.local, "device_images", False)
        half = self.geom.local_strides // 2
        k = half
        if hasattr(self.local, "image_bytes") and self.exchange_chunk_bytes:
            per = max(1, self.local.image_bytes(qb, send_bit) // max(1, half))
            k = max(1, min(half, self.exchange_chunk_bytes // per))
        k = min(self.comm.allgather(k))  # every rank streams the same number of chunks
        for first in range(0, half, k):
            payload = self.local.pack(qb, send_bit, first, k)
            got = self.comm.exchange(peer, payload, device=device)
            self.local.unpack(got, 1 << qb)
        self.exchanges += 1

    def _make_local(self, p: int, keep: Optional[int], index: int) -> int:
        """Physical local position of logical stride bit p, swapping it in from a
        rank bit if needed (evicting the least recently used local bit other
        than `keep`)."""
        g = self.geom
        nloc = g.local_qubits - g.stride_bits
        q = self.pi[p]
        if q < nloc:
            return q
        cands = [v for v in range(nloc) if v != keep]
        if not cands:
            # the control holds the only local stride bit: evict it -- it becomes a
            # rank bit, and a control on a rank bit is the rank-level skip
            cands = list(range(nloc))
        if self.next_target is not None:
            v = max(cands, key=lambda v: (self._next_use(self.inv[v], index), -v))
        else:
            v = min(cands, key=lambda v: (self.last_use[self.inv[v]], v))
        self._swap(q - nloc, v)
        pv = self.inv[v]
        self.pi[p], self.pi[pv] = v, q
        self.inv[v], self.inv[q] = p, pv
        return v

    def apply_gate(self, gate: GateOp, ladder: Sequence[float], theta: float, index: int = 0):
        g = self.geom
        Q, s = g.local_qubits, g.stride_bits
        nloc = Q - s
        gate.validate(g.n_qubits)
        pair_bit_global = None
        reports: List[tuple] = []
        if gate.kind in (KIND_SINGLE, KIND_CONTROLLED):
            t, c = gate.target, gate.control
            ctl_phys = None  # physical stride position of a stride-bit control
            if gate.kind == KIND_CONTROLLED and c >= s:
                ctl_phys = self.pi[c - s]
            lt = t
            if t >= s:
                pair_bit_global = 1 << (t - s)
                keep = ctl_phys if (ctl_phys is not None and ctl_phys < nloc) else None
                lt = s + self._make_local(t - s, keep, index)
                self.last_use[t - s] = index
                if ctl_phys is not None:
                    ctl_phys = self.pi[c - s]
            participate = True
            local = GateOp(gate.kind, gate.unitary, lt, c, 0, gate.phase_theta, gate.label)
            if ctl_phys is not None:
                if ctl_phys >= nloc:  # control on a rank bit: the rank applies it or nothing
                    participate = bool((self.r >> (ctl_phys - nloc)) & 1)
                    local = GateOp.single(gate.unitary, lt, gate.label)
                else:
                    local.control = s + ctl_phys
                self.last_use[c - s] = index
            if participate:
                reports = self.local.apply(local, ladder, theta)
        elif gate.kind == KIND_FLIP:
            jp = self._log_to_phys(gate.flip_index >> s)
            if (jp >> nloc) == self.r:
                off = ((jp & ((1 << nloc) - 1)) << s) | (gate.flip_index & ((1 << s) - 1))
                reports = self.local.apply(GateOp.phase_flip(off), ladder, theta)
        else:
            # mean pass (aalc.cpp:270-295): per-stride sums, combined serially
            # in LOGICAL global stride order, divided by the amplitude count
            parts = self.comm.allgather(self.local.stride_sums().tobytes())
            allp = np.concatenate([np.frombuffer(p).reshape(-1, 2) for p in parts])
            order = self._logical_order()
            sr = si = 0.0
            for re_, im_ in allp[order].tolist():
                sr += re_
                si += im_
            na = float(1 << g.n_qubits)
            reports = self.local.apply(gate, ladder, theta, mean=(sr / na, si / na))
        # one gather per gate: this rank's reports keyed by LOGICAL global unit
        # order (reference: ascending lo stride; a pair unit reports lo then hi)
        # and its per-stride (scale, sum_sq)
        nsl = g.local_strides
        buf = np.zeros((nsl + 1, 10))
        rep = np.asarray(reports, dtype=np.float64).reshape(-1, 6)
        buf[0, 0] = len(rep)
        if len(rep):
            gj = self._phys_to_log(self.r * nsl + rep[:, 0].astype(np.int64))
            if pair_bit_global is not None:
                k0, k1 = gj & ~pair_bit_global, (gj & pair_bit_global) != 0
            else:
                k0, k1 = gj, np.zeros(len(gj))
            buf[1:1 + len(rep), 0] = k0
            buf[1:1 + len(rep), 1] = k1
            buf[1:1 + len(rep), 2] = gj
            buf[1:1 + len(rep), 3:8] = rep[:, 1:6]
        sc, sm = self.local.stride_norms()
        buf[1:, 8] = sc
        buf[1:, 9] = sm
        parts = self.comm.allgather_array(buf)
        # global renormalisation, serial in LOGICAL global stride order
        # (aalc.cpp:410-419); np.cumsum is a sequential left-to-right fold
        scales = np.concatenate([p_[1:, 8] for p_ in parts])
        sums = np.concatenate([p_[1:, 9] for p_ in parts])
        order = self._logical_order()
        scales, sums = scales[order], sums[order]
        total = float(np.cumsum(scales * scales * sums)[-1])
        if total > 0.0:
            f = 1.0 / math.sqrt(total)
            self.local.scale_all(f)
            scales = scales * f
        nsq = float(np.cumsum(scales * scales * sums)[-1])
        self.norm_sq = nsq
        # GateRecord fold in global unit order (aalc.cpp:612-631)
        rows = np.concatenate([p_[1:1 + int(p_[0, 0]), :8] for p_ in parts])
        rows = rows[np.lexsort((rows[:, 1], rows[:, 0]))]
        rec = GateRecord(gate_index=index, gate_label=gate.label, stride_count=len(rows))
        rec.min_ratio = float(rows[:, 4].min()) if len(rows) else math.inf
        rec.mean_ratio = float(np.cumsum(rows[:, 4])[-1]) / len(rows) if len(rows) else 0.0
        rec.max_chosen_delta = max(0.0, float(rows[:, 3].max())) if len(rows) else 0.0
        rec.bytes_before = int(rows[:, 5].sum())
        rec.bytes_after = int(rows[:, 6].sum())
        rec.norm_after = math.sqrt(nsq)
        viol = int((rows[:, 7] == 0.0).sum())
        return rec, viol

    def amplitudes(self) -> np.ndarray:
        """Whole LOGICAL state on every rank (small states only; for tests)."""
        g = self.geom
        L = 1 << g.stride_bits
        parts = self.comm.allgather(self.local.amplitudes().tobytes())
        phys = np.concatenate([np.frombuffer(p, dtype=np.complex128) for p in parts]).reshape(-1, L)
        out = np.empty_like(phys)
        out[self._phys_to_log(np.arange(len(phys), dtype=np.int64))] = phys
        return out.reshape(-1)


def run_sharded(program, geom: ShardGeometry, comm, backend, basis: int, ladder, theta):
    """run_program over a sharded state; returns (state, records, violations)."""
    st = ShardedState(geom, comm, backend, basis)
    st.set_schedule(program.gates)
    recs = []
    viol = 0
    for i, g in enumerate(program.gates):
        rec, v = st.apply_gate(g, ladder, theta, i)
        recs.append(rec)
        viol += v
    return st, recs, viol


def run_thread_cluster(program, geom: ShardGeometry, backend_factory, basis: int, ladder, theta):
    """All ranks as threads of this process (ThreadComm); returns
    (amplitudes, records of rank 0)."""
    size = 1 << geom.rank_bits
    grp = ThreadGroup(size)
    out = [None] * size
    errs = []

    def worker(r):
        try:
            st, recs, _ = run_sharded(program, geom, ThreadComm(grp, r), backend_factory(r), basis,
                                      ladder, theta)
            out[r] = (st.amplitudes(), recs)
        except BaseException as e:  # surface worker failures
            errs.append(e)
            grp.barrier.abort()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out[0]


def plan_exchanges(program, geom: ShardGeometry, belady: bool = True) -> List[int]:
    """Gate indices at which the lazy qubit permutation exchanges strides
    between partner ranks, for `program` on `geom` — the same decisions
    ShardedState makes, without any data (for sizing multi-GPU runs, e.g.
    BASELINE's 37-qubit QFT on 8 GPUs)."""

    class _Plan(ShardedState):
        def __init__(self):  # no communicator, no local engine
            self.geom, self.r = geom, 0
            nb = geom.n_qubits - geom.stride_bits
            self.pi, self.inv = list(range(nb)), list(range(nb))
            self.last_use = [-1] * nb
            self.exchanges = 0
            self.next_target = None
            self.at = []

        def _swap(self, b, qb):
            self.exchanges += 1

    st = _Plan()
    if belady:
        st.set_schedule(program.gates)
    s = geom.stride_bits
    out = []
    for i, g in enumerate(program.gates):
        if g.kind in (KIND_SINGLE, KIND_CONTROLLED) and g.target >= s:
            ctl = st.pi[g.control - s] if (g.kind == KIND_CONTROLLED and g.control >= s) else None
            nloc = geom.local_qubits - s
            before = st.exchanges
            st._make_local(g.target - s, ctl if (ctl is not None and ctl < nloc) else None, i)
            st.last_use[g.target - s] = i
            if g.kind == KIND_CONTROLLED and g.control >= s:
                st.last_use[g.control - s] = i
            if st.exchanges != before:
                out.append(i)
    return out
