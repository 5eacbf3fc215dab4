"""CPU-side checks of the C ABI: the library builds, loads and exports every symbol
include/jdob.h declares; host-only helpers work; argument errors are reported
without touching a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2504_14611_b200 import build
    build.build()
    import paper_2504_14611_b200 as J
    return J.lib()


def declared_symbols():
    h = open(os.path.join(ROOT, "include", "jdob.h")).read()
    return sorted(set(re.findall(r"JDOB_API\s+[\w\s\*]+?\b(jdob_\w+)\s*\(", h)))


def test_header_symbols_exported(L):
    syms = declared_symbols()
    assert len(syms) == 18, syms
    assert set(syms) == set(__import__("paper_2504_14611_b200").EXPORTED), syms
    for s in syms:
        assert hasattr(L, s), s
    import paper_2504_14611_b200 as J
    assert sorted(J.EXPORTED) == syms


def test_version_and_error(L):
    assert b"sm_100a" in L.jdob_version()
    assert L.jdob_last_error() == b""


def test_bf_space_size(L):
    import paper_2504_14611_b200 as J
    assert J.bf_space_size(0, 11, 8, 64) == 12 ** 8 * 64 == 27_518_828_544
    assert J.bf_space_size(1, 11, 8, 64) == 12 * 256 * 64 == 196_608
    assert J.bf_space_size(0, 63, 11, 64) == 0          # >= 2^62 -> 0
    assert J.bf_space_size(0, 4, 2, 3) == 75            # C1: 5^2 * 3
    assert J.bf_space_size(1, 4, 2, 3) == 60            # C1: 5 * 4 * 3


def test_workspace_bytes_host_only(L):
    import paper_2504_14611_b200._binding as B
    ms = (B.JModel * 2)(B.JModel(4, 2), B.JModel(19, 32))
    assert L.jdob_workspace_bytes(ms, 2, 0) > 0
    assert L.jdob_workspace_bytes(ms, 2, 1) > 0
    bad = (B.JModel * 1)(B.JModel(0, 2))
    assert L.jdob_workspace_bytes(bad, 1, 0) == 0
    assert L.jdob_workspace_bytes(ms, 2, 7) == 0


def test_argument_errors_without_gpu(L):
    import paper_2504_14611_b200._binding as B
    ms = (B.JModel * 1)(B.JModel(4, 2))             # NULL tables
    b = B.JBatch()
    r = B.JResult()
    assert L.jdob_solve_batch(ms, 1, C.byref(b), 0, C.byref(r), None, 0, None) == B.EINVAL
    assert b"NULL" in L.jdob_last_error()
    assert L.jdob_solve_batch(None, 0, None, 0, None, None, 0, None) == B.EINVAL
    assert L.jdob_bruteforce(ms, 1, C.byref(b), 0, 0, 1, None, None, None, None, None, 0, None) == B.EINVAL
    # the entry points added in round 2 reject bad arguments on the host, before any CUDA call
    r3 = (B.JResult * 3)()
    assert L.jdob_solve_batch_modes(ms, 1, C.byref(b), r3, None, 0, None) == B.EINVAL
    assert L.jdob_solve_batch_modes(None, 0, None, None, None, 0, None) == B.EINVAL
    sb = B.JSharedBatch()
    assert L.jdob_solve_shared_host(ms, 1, C.byref(sb), 0, C.byref(r), None, None, None) == B.EINVAL
    assert L.jdob_solve_shared_host(ms, 1, None, 0, C.byref(r), None, None, None) == B.EINVAL
    assert L.jdob_stats(None, None, None, 0, None) == B.EINVAL
    assert L.jdob_stats_part(C.byref(b), C.byref(r), 10, 3, 0, None, 0, None) == B.EINVAL   # NULL stats
    gp = B.JGenParams()
    n_users = C.c_int64()
    assert L.jdob_generate_c5_instances(C.byref(gp), C.byref(b), None, None, 0, None) == B.EINVAL
    b5 = B.JBatch(5, 1)
    assert L.jdob_generate_c5_instances(C.byref(gp), C.byref(b5), C.byref(n_users), None, 0, None) == B.EINVAL
    assert L.jdob_generate_workspace_bytes(-1) == 0
    assert L.jdob_workspace_bytes(None, 0, 2) > 0          # jdob_stats needs no model part


def test_no_cpu_fallback():
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_2504_14611_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "jdob_oracle" not in src, f


def test_oracle_header_independent():
    # the oracle shares no header with the CUDA path
    src = open(os.path.join(ROOT, "oracle", "jdob_oracle.c")).read()
    assert "#include \"" not in src
    assert "jdob.h" not in src


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of jdob_model / jdob_batch / jdob_result / jdob_grouped_result have the
    header's field offsets and sizes (compiled with the system C compiler against include/jdob.h)."""
    import shutil
    import subprocess

    from paper_2504_14611_b200 import _binding as B
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"jdob_model": B.JModel, "jdob_batch": B.JBatch, "jdob_result": B.JResult,
               "jdob_grouped_result": B.JGrouped, "jdob_gen_params": B.JGenParams,
               "jdob_shared_batch": B.JSharedBatch}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "jdob.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    inc = os.path.join(ROOT, "include")
    subprocess.run([cc, "-I", inc, str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            c, f, v = ln.split()
            got[(c, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
