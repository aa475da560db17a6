"""Gate-by-gate GPU vs oracle diagnostic (run on the GPU box)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import circuit as cc
from oracle import Oracle
from helpers import golden_runs, golden_program

def serial_sum(re, im):
    s = 0.0
    for a, b in zip(re.tolist(), im.tolist()):
        s = s + (a * a + b * b)
    return s

def run(name=None, prog=None, s=None, basis=0, ladder=None, theta=1.0, maxg=10**9):
    o = Oracle()
    if name:
        e = golden_runs()[name]; prog = golden_program(e); s = e["stride_bits"]; basis = e["basis"]; ladder = e["ladder"]; theta = e["theta"]
    n = prog.n_qubits
    st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), basis)
    ost = o.state(n, s, basis)
    lad = q.ErrorBoundLadder.make(ladder)
    for gi, g in enumerate(prog.gates[:maxg]):
        r = st.apply_gate(g, lad, q.RatioThreshold(theta))
        orr, on = ost.apply_gate(g, ladder, theta)
        bad = []
        for j in range(1 << (n - s)):
            b, sc, ss = st.export_blocks(j)
            ob = ost.export_blocks(j)
            osc, oss, _, _ = ost.stride_info(j)
            if b != ob or sc != osc or ss != oss:
                bad.append((j, b == ob, sc, osc, ss, oss))
        if bad or r.norm_after != on:
            print(f"gate {gi} {g.label}: norm {r.norm_after!r} vs {on!r}; {len(bad)} strides differ")
            for (j, same_b, sc, osc, ss, oss) in bad[:4]:
                re, im = st.stored_stride(j)
                print(f"  stride {j}: blocks_equal={same_b} scale {sc!r}/{osc!r} sum {ss!r}/{oss!r} serial(gpu stored)={serial_sum(re, im)!r}")
                if not same_b:
                    b, _, _ = st.export_blocks(j); ob = ost.export_blocks(j)
                    k = next((i for i, (x, y) in enumerate(zip(b, ob)) if x != y), min(len(b), len(ob)))
                    print(f"    len {len(b)} vs {len(ob)} first diff byte {k}: gpu {b[k:k+12].hex()} oracle {ob[k:k+12].hex()}")
            return
    print(name or "case", "all gates identical")



def sum_probe():
    """Run the failing case to gate 55, dump stride 1 stored values, and
    re-sum them with the device hook."""
    import ctypes as C
    from paper_1811_05140_b200.engine import lib
    e = golden_runs()["grover12_gates_pow2"]
    prog = golden_program(e)
    n, s = prog.n_qubits, e["stride_bits"]
    st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), e["basis"])
    lad = q.ErrorBoundLadder.make(e["ladder"])
    for g in prog.gates[:56]:
        st.apply_gate(g, lad, q.RatioThreshold(1.0))
    re, im = st.stored_stride(1)
    np.save(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "stride1.npy"), np.stack([re, im]))
    out = C.c_double()
    lib().qcs_debug_stride_sumsq.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_double)]
    rc = lib().qcs_debug_stride_sumsq(re.ctypes.data, im.ctypes.data, re.size, C.byref(out))
    print("hook rc", rc, "device", repr(out.value), "serial", repr(serial_sum(re, im)), "engine", st.stride_info(1)[1])


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        if nm == "sum_probe":
            sum_probe()
        else:
            run(nm)
