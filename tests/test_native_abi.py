"""The C-ABI library loads, exports every symbol of include/mapple_b200.h, and
its code generator + NVRTC produce sm_100a cubins (no GPU needed)."""

import re
from pathlib import Path

import pytest

from conftest import ROOT, mapping_cases
from paper_2507_17087_b200 import native
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.spaces import MachineShape

HEADER = ROOT / "include" / "mapple_b200.h"


def _declared():
    text = HEADER.read_text()
    decl = r"^(?:int|void|size_t|const char\s*\*)\s+(pm_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_every_declared_symbol_is_exported():
    lib = native.lib()
    declared = _declared()
    assert declared, "no pm_* declarations found"
    for name in declared:
        assert hasattr(lib, name), name
        assert name in native.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.pm_abi_version() == native.ABI_VERSION


def test_opcodes_match_header():
    from paper_2507_17087_b200.dsl import lower as L

    text = HEADER.read_text()
    for i, name in enumerate(L.OP_NAMES):
        m = re.search(rf"PM_OP_{name}\s*=\s*(\d+)", text)
        assert m and int(m.group(1)) == i, name


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", str(native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("case", [c for c in mapping_cases()[:: 37] if isinstance(c["table"], list)])
def test_codegen_compiles_with_nvrtc(case):
    prog = parse(case["source"])
    fn = compile_mapper(prog, case["task"], MachineShape("GPU", *case["machine"]))
    for implicit in (True, False):
        pp = fn.program_for(case["ispace"], implicit=implicit, k=len(case["ispace"]))
        src = pp.source()
        assert "pm_map_points" in src
        pp.compile_check()
        pp.compile_check_fused()
        pp.compile_check_probe()


def test_failure_probes_compile_for_message_sites():
    """Every golden program whose failures quote per-point values has a probe
    that NVRTC accepts (the GPU run formats the messages from it)."""
    done = 0
    for case in mapping_cases():
        if not isinstance(case["table"], list) or not any(
                isinstance(r, dict) and "index" in r["message"] for r in case["table"]):
            continue
        fn = compile_mapper(parse(case["source"]), case["task"],
                            MachineShape("GPU", *case["machine"]))
        pp = fn.program_for(case["ispace"], implicit=True)
        if pp.lowered.program.site_fmts:
            pp.compile_check_probe()
            done += 1
        if done >= 6:
            break
    assert done >= 1


def test_bad_program_is_rejected():
    import ctypes

    bad = native.PmInsn(99, 0, 0, 0, 0, -1, 0, 0)
    insns = (native.PmInsn * 1)(bad)
    widths = (ctypes.c_uint8 * 1)(0)
    ext = (ctypes.c_int64 * 1)(1)
    prog = native.PmProgram(1, insns, 1, widths, 1, 1, ext)
    rc = native.lib().pm_compile_check(ctypes.byref(prog))
    assert rc == 1
    assert b"opcode" in native.lib().pm_last_error()


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    fn = compile_mapper(parse(Path(ROOT / "tests" / "golden" / "make_golden.py").read_text()
                              [:0] + "m = Machine(GPU)\ndef f(Tuple p, Tuple s):\n"
                              "    return m[0, 0]\nIndexTaskMap t f\n"), "t",
                        MachineShape("GPU", 1, 1))
    with pytest.raises(native.NativeError):
        fn.map_ispace((4,))


def _c_layout(struct, fields):
    """sizeof + offsetof of a header struct, from a C program compiled with gcc."""
    import shutil
    import subprocess
    import tempfile

    if not shutil.which("gcc"):
        pytest.skip("gcc is absent")
    body = "".join(f'printf("%zu ", offsetof({struct}, {f}));' for f in fields)
    src = ("#include <stdio.h>\n#include <stddef.h>\n#include \"mapple_b200.h\"\n"
           f"int main(void){{printf(\"%zu \", sizeof({struct}));{body}return 0;}}\n")
    with tempfile.TemporaryDirectory() as d:
        c, exe = Path(d) / "l.c", Path(d) / "l"
        c.write_text(src)
        subprocess.run(["gcc", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
                        str(c), "-o", str(exe)], check=True, capture_output=True)
        return [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                               check=True).stdout.split()]


def test_ctypes_structs_match_the_header_layout():
    """Every view struct the Python side builds has the C header's size and offsets
    (the stencil / hydro views and the step ops changed shape in round 2)."""
    import ctypes

    from paper_2507_17087_b200.executors.circuit import PmCircuitView
    from paper_2507_17087_b200.executors.hydro import PmHydroView
    from paper_2507_17087_b200.executors.stencil import PmStencilView
    from paper_2507_17087_b200.peer import PmPeerBarrierView, PmPeerCopy, PmStepOp

    renames = {"in_": "in"}
    for struct, cls in (("pm_step_op", PmStepOp), ("pm_stencil_view", PmStencilView),
                        ("pm_hydro_view", PmHydroView), ("pm_circuit_view", PmCircuitView),
                        ("pm_peer_barrier_view", PmPeerBarrierView),
                        ("pm_peer_copy", PmPeerCopy), ("pm_program", native.PmProgram),
                        ("pm_insn", native.PmInsn)):
        names = [f[0] for f in cls._fields_]
        want = _c_layout(struct, [renames.get(n, n) for n in names])
        got = [ctypes.sizeof(cls)] + [getattr(cls, n).offset for n in names]
        assert got == want, (struct, list(zip(["sizeof"] + names, got, want)))


def test_step_op_kinds_match_the_header():
    """peer.py's step-op kinds are the header's PM_STEP_* values, and pm_steps_create
    rejects an unknown kind before touching the GPU."""
    import ctypes
    import re

    from paper_2507_17087_b200 import peer

    hdr = (ROOT / "include" / "mapple_b200.h").read_text()
    enum = dict((k, int(v)) for k, v in re.findall(r"PM_STEP_(\w+) = (\d+)", hdr))
    for name in ("PULL", "WAIT", "GEMM_BF16", "GEMM_TF32", "MEMSET", "BARRIER",
                 "COPY_BARRIER", "FORK"):
        assert getattr(peer, name) == enum[name], name
    assert peer.LANES == int(re.search(r"#define PM_STEP_LANES (\d+)", hdr).group(1))
    lib = native.lib()
    bad = (peer.PmStepOp * 1)(peer.PmStepOp(kind=99))
    out = ctypes.c_void_p()
    assert lib.pm_steps_create(bad, 1, ctypes.byref(out)) != 0
    assert b"unknown kind" in lib.pm_last_error()
