"""SASS summary of the objective kernels (developer tool, no GPU needed):
nvcc -cubin of the kernel template with the C2 / Eq. 6 theory (the AOT check
_build.aot_check() writes), then per entry point: ptxas registers / spills and
static instruction-class counts (FP64, TMA, mbarrier, shared/global memory).

    python tools/sass_summary.py > profiles/<round>_sass_summary.txt
"""
import re, subprocess, sys
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_02334_b200 import _build  # noqa: E402

ENTRIES = ["musr_chi2_c32", "musr_chi2_c32big", "musr_chi2_f64", "musr_mlh_c32", "musr_mlh_f64",
           "musr_chi2_c32_batch", "musr_mlh_c32_batch"]
CLASSES = {"FP64": ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"), "TMA bulk copy": ("UBLKCP",),
           "mbarrier/SYNCS": ("SYNCS",), "shared load": ("LDS",), "shared store": ("STS",),
           "global load": ("LDG", "LD"), "global store": ("STG", "ST"), "local (spill)": ("LDL", "STL"),
           "MUFU": ("MUFU",), "conversion": ("F2F", "I2F", "F2I"), "atomic": ("ATOMG", "ATOM", "RED", "REDG"),
           "shuffle": ("SHFL",)}

cubin = _build.aot_check()
log = subprocess.run([_build.NVCC, *_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
                      "-cubin", "-Xptxas", "-v", "-I", str(_build.CSRC), "-o", "/dev/null",
                      str(cubin.with_suffix(".cu"))], capture_output=True, text=True).stderr
regs = dict(re.findall(r"Function properties for (\w+)\n\s+(.*?)\n", log))
used = dict(re.findall(r"Compiling entry function '(\w+)'.*?\nptxas info\s+: Function properties.*?\n.*?\n"
                       r"ptxas info\s+: Used (\d+) registers", log, re.S))
print(f"# SASS summary: {cubin.name} (C2 / Eq. 6 theory), nvcc sm_100a, static instruction counts")
for e in ENTRIES:
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", e, str(cubin)], capture_output=True,
                          text=True).stdout
    ops = Counter(m.split(".")[0] for m in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", sass))
    print(f"\n## {e}: {used.get(e, '?')} registers; {regs.get(e, '?')}")
    print("  total " + str(sum(ops.values())) + "; " + "; ".join(
        f"{k} {sum(ops[x] for x in v)}" for k, v in CLASSES.items()))
