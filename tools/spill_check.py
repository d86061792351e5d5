"""Compile the kernel template for every workload theory (nvcc, sm_100a) and
report registers / spills per entry point (developer tool, no GPU)."""
import re, subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_02334_b200 import _build, workloads as W
from paper_1604_02334_b200.codegen import lower
from paper_1604_02334_b200.theory import parse

extra = sys.argv[1:]
for name in ("C1", "C2", "C3"):
    w = W.WORKLOADS[name]()
    frag = lower(parse(w.expr.source).ast).source
    cu = _build.BUILD / f"spill_{name}.cu"
    _build.BUILD.mkdir(exist_ok=True)
    cu.write_text('#include "musr_prelude.cuh"\n' + frag + '\n#include "musr_kernel.cuh"\n')
    out = subprocess.run([_build.NVCC, *_build.ARCH, "-O3", "-std=c++17", "--fmad=false", "-cubin",
                          "-Xptxas", "-v", "-I", str(_build.CSRC), *extra, "-o", "/dev/null", str(cu)],
                         capture_output=True, text=True).stderr
    res = []
    for m in re.finditer(r"Function properties for (musr_\w+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n.*?Used (\d+) registers", out):
        fn, st, ss, sl, regs = m.groups()
        if fn.startswith(("musr_chi2", "musr_mlh")):
            res.append(f"{fn[5:]}:{regs}r" + (f"/SPILL{ss}" if int(ss) else ""))
    print(name, " ".join(res))
