"""SASS instruction summary of every kernel in libmapple_b200.so (and of the NVRTC
point programs K1 / fused K1+K2 / failure probe for a sample mapper): per kernel,
counts of the instruction classes that show what the code runs on (tcgen05 MMA,
TMA, TMEM loads, global / shared memory, atomics, shuffles), plus registers.

    python tools/sass_summary.py > profiles/r02_sass_summary.txt

Runs without a GPU (cuobjdump on the built library; NVRTC cubins via
PM_DUMP_CUBIN from the compile-check entry points).
"""

import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CLASSES = OrderedDict([
    ("UTCHMMA/UTCQMMA (tcgen05.mma)", r"^UTC[HQ]?MMA|^UTCMMA"),
    ("UTMALDG (TMA load)", r"^UTMALDG"),
    ("UTMASTG (TMA store)", r"^UTMASTG"),
    ("UTMAREDG (TMA reduce)", r"^UTMAREDG"),
    ("UBLKCP (bulk copy)", r"^UBLKCP"),
    ("LDTM/STTM (TMEM)", r"^(LDTM|STTM)"),
    ("LDG", r"^LDG"),
    ("STG", r"^STG"),
    ("LDS", r"^LDS"),
    ("STS", r"^STS"),
    ("ATOM/RED (global)", r"^(ATOMG|RED|ATOM\b)"),
    ("ATOMS (shared)", r"^ATOMS"),
    ("SHFL", r"^SHFL"),
    ("VOTE/MATCH", r"^(VOTE|MATCH)"),
    ("BAR/SYNCS", r"^(BAR|SYNCS)"),
    ("FFMA/FADD/FMUL", r"^(FFMA|FADD|FMUL)"),
    ("IMAD/IADD3", r"^(IMAD|IADD3)"),
    ("total", r"."),
])


def sass_of(cubin_or_so: str) -> dict:
    out = subprocess.run(["cuobjdump", "-sass", cubin_or_so], capture_output=True, text=True).stdout
    kernels, cur = OrderedDict(), None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = kernels.setdefault(m.group(1), Counter())
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur is not None:
            op = m.group(1)
            for name, pat in CLASSES.items():
                if re.match(pat, op):
                    cur[name] += 1
    return kernels


def regs_of(path: str) -> dict:
    out = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    regs, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+)", line)
        if m and cur:
            regs[cur] = int(m.group(1))
    return regs


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines()


def report(title, path):
    ks = sass_of(path)
    regs = regs_of(path)
    pretty = demangle(list(ks))
    print(f"## {title}: {path}\n")
    for (name, cnt), nice in zip(ks.items(), pretty):
        nice = nice.replace("(anonymous namespace)::", "")
        nice = re.sub(r"\(.*", "", nice)[:110]
        parts = [f"{k.split(' ')[0]}={v}" for k, v in cnt.items() if v and k != "total"]
        print(f"{nice}  [regs {regs.get(name, '?')}, {cnt['total']} instructions]")
        print("    " + ", ".join(parts))
    print()


def main():
    lib = ROOT / "paper_2507_17087_b200" / "libmapple_b200.so"
    report("libmapple_b200.so (nvcc, sm_100a)", str(lib))
    # NVRTC point programs of the stencil's decompose block mapper (8 processors)
    from paper_2507_17087_b200.dsl import compile_mapper, parse
    from paper_2507_17087_b200.spaces import MachineShape

    src = ("m = Machine(GPU)\ndef blk(Tuple p, Tuple s):\n"
           "    q = m.merge(0, 1).decompose(0, s)\n    return q[*(p * q.size / s)]\n"
           "IndexTaskMap t blk\n")
    fn = compile_mapper(parse(src), "t", MachineShape("GPU", 1, 8))
    pp = fn.program_for((32768, 32768), implicit=True)
    with tempfile.TemporaryDirectory() as d:
        for name, call in (("K1 pm_map_points", pp.compile_check),
                           ("fused K1+K2 (pm_map_hist / pm_map_scatter)", pp.compile_check_fused),
                           ("failure probe", pp.compile_check_probe)):
            path = os.path.join(d, "k.cubin")
            os.environ["PM_DUMP_CUBIN"] = path
            call()
            os.environ.pop("PM_DUMP_CUBIN")
            report(f"NVRTC {name}, 32768^2 launch, decompose block mapper", path)


if __name__ == "__main__":
    main()
