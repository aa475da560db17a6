"""The C++ façade (include/qcs_b200.hpp) in the reference's own types.

CPU: the header compiles against the reference's headers (when the reference
is mounted, i.e. in the build container).  GPU: oracle/_ref/facade_parity —
the façade + the unmodified reference library, built by oracle/Makefile —
runs the same programs through qcs::run_program and qcs::b200::run_program
and compares every record, amplitude, stored stride, checkpoint byte and
codec block (tests/cpp/facade_parity.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
BIN = os.path.join(ROOT, "oracle", "_ref", "facade_parity")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not mounted")
def test_facade_header_compiles():
    subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-Wall", "-Wextra", "-I", REF_INC,
                    "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "facade_parity.cpp")],
                   check=True)


@pytest.mark.gpu
def test_facade_parity_against_reference():
    if not os.path.exists(BIN):
        pytest.skip("facade_parity not built (needs the reference sources at build time)")
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "circuits")], capture_output=True,
                       text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") >= 11 and "0 failure(s)" in r.stdout


ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.gpu
def test_reference_acceptance_suite_on_b200():
    """The reference's UNMODIFIED acceptance suite (proj/tests/acceptance.cpp,
    11 criteria) linked to the B200 engine through the
    link-level drop-in (include/qcs_b200_dropin.hpp +
    paper_1811_05140_b200/host/qcs_b200_dropin.cpp) instead of the reference's
    aalc.cpp and codec.cpp."""
    if not os.path.exists(ACC):
        pytest.skip("acceptance_b200 not built (needs the reference sources at build time)")
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=900, cwd="/tmp")
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "11 of 11 criteria passed" in r.stdout


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not mounted")
def test_dropin_objects_replace_engine_and_codec():
    """acceptance_b200 defines the engine/codec symbols from the drop-in object
    (not the reference's aalc.o / codec.o) and loads libqcs_b200.so."""
    if not os.path.exists(ACC):
        pytest.skip("acceptance_b200 not built")
    nm = subprocess.run(["nm", "-C", ACC], capture_output=True, text=True).stdout
    for sym in ("qcs::compress_lossy(", "qcs::CompressedState::apply_gate(", "qcs::run_program("):
        assert any(sym in l and " T " in l for l in nm.splitlines()), sym
    assert "libqcs_b200.so" in subprocess.run(["ldd", ACC], capture_output=True, text=True).stdout
