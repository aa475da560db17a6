"""Closed-form QFT stage states on the device (benchmark / test setup).

circuit.qft_stage gives the exact state build_qft(n) (circuit.cpp:274-297)
holds after any gate; circuit.stage_tables factors it for stride-by-stride
generation.  This module generates those amplitudes with torch on the GPU and
compresses them into a CompressedState through qcs_load_strides_device, and
measures a state's fidelity against them.  Setup and checking only: nothing
here is on the timed path.
"""
from __future__ import annotations

import math

from . import circuit as cc


class StageGen:
    """Device generator of a closed-form stage state (circuit.stage_tables):
    t = hr*lr - hi*li, u = hr*li + hi*lr, (amp*t, amp*u), +0.0 where the
    unprocessed qubits disagree with the basis -- one IEEE operation per torch
    kernel, the same operations in the same order as the reference arm's C++
    generator (oracle/ref_capi.cpp ref_state_from_tables)."""

    def __init__(self, tables, n, s, device):
        import torch
        f = lambda a: torch.from_numpy(a).to(device)  # noqa: E731
        self.lr, self.li, self.hr, self.hi = (f(tables[k]) for k in ("lo_re", "lo_im", "hi_re", "hi_im"))
        self.amp = tables["amp"]
        L, NS = 1 << s, 1 << (n - s)
        zm, zv = tables["zmask"], tables["zval"]
        e = torch.arange(L, dtype=torch.int64, device=device)
        j = torch.arange(NS, dtype=torch.int64, device=device)
        self.mlo = (e & (zm & (L - 1))) == (zv & (L - 1))
        self.mhi = (j & (zm >> s)) == (zv >> s)
        self.zero = torch.zeros((), dtype=torch.float64, device=device)

    def fill(self, v, j0, m):
        """v: [m, 2, L] float64 view for strides [j0, j0 + m)."""
        import torch
        hr, hi = self.hr[j0:j0 + m, None], self.hi[j0:j0 + m, None]
        mask = self.mhi[j0:j0 + m, None] & self.mlo[None, :]
        t = torch.sub(torch.mul(hr, self.lr), torch.mul(hi, self.li))
        torch.where(mask, torch.mul(t, self.amp), self.zero, out=v[:, 0, :])
        del t
        u = torch.add(torch.mul(hr, self.li), torch.mul(hi, self.lr))
        torch.where(mask, torch.mul(u, self.amp), self.zero, out=v[:, 1, :])


def load_stage_state(q, n, s, x, g, lad, th, device, batch=64):
    """basis_state + the closed-form state after gate g, compressed stride batch
    by stride batch through qcs_load_strides_device (untimed setup)."""
    import torch
    geom = q.StateGeometry.make(n, s)
    st = q.CompressedState.basis_state(geom, x, device=device)
    gen = StageGen(cc.stage_tables(n, s, *cc.qft_stage(n, x, g)), n, s, device)
    NS, L = geom.n_strides(), geom.stride_len()
    batch = min(batch, NS)
    buf = torch.empty(batch * 2 * L, dtype=torch.float64, device=device)
    for j0 in range(0, NS, batch):
        m = min(batch, NS - j0)
        gen.fill(buf[: m * 2 * L].view(m, 2, L), j0, m)
        torch.cuda.synchronize()          # the engine runs on its own stream
        st.load_strides_device(j0, m, buf.data_ptr(), lad, th)
    del buf, gen
    return st


def stage_fidelity(st, n, s, x, g, device, batch=64):
    """Fidelity |<e|a>| / (|e| |a|) (dense.cpp:94-108) of the state against the
    exact closed-form state after gate g, streamed stride batch by batch; also
    the largest amplitude error."""
    import torch
    gen = StageGen(cc.stage_tables(n, s, *cc.qft_stage(n, x, g)), n, s, device)
    L, NS = 1 << s, 1 << (n - s)
    batch = min(batch, NS)
    a = torch.empty(batch * 2 * L, dtype=torch.float64, device=device)
    e = torch.empty_like(a)
    ov_r = ov_i = na = ne = 0.0
    maxerr = 0.0
    for j0 in range(0, NS, batch):
        m = min(batch, NS - j0)
        av, ev = a[: m * 2 * L].view(m, 2, L), e[: m * 2 * L].view(m, 2, L)
        st.read_strides_device(j0, m, a.data_ptr())
        gen.fill(ev, j0, m)
        ar, ai, er, ei = av[:, 0], av[:, 1], ev[:, 0], ev[:, 1]
        ov_r += float(torch.sum(er * ar + ei * ai))
        ov_i += float(torch.sum(er * ai - ei * ar))
        na += float(torch.sum(ar * ar + ai * ai))
        ne += float(torch.sum(er * er + ei * ei))
        maxerr = max(maxerr, float(torch.max(torch.abs(av - ev))))
    return math.hypot(ov_r, ov_i) / math.sqrt(na * ne), maxerr
