"""SASS summary of the objective kernels as the product builds them (developer
tool, no GPU needed): the library's NVRTC compile of the C2 / Eq. 6 theory
(musr_compile_theory with MUSR_DUMP_CUBIN and ptxas -v), then per entry point:
registers / spills and static instruction-class counts (FP64, TMA, mbarrier,
shared/global memory).

    python tools/sass_summary.py > profiles/<round>_sass_summary.txt
"""
import ctypes as C, os, re, subprocess, sys, tempfile
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
cub = Path(tempfile.mkdtemp()) / "musr_theory.cubin"
os.environ["MUSR_DUMP_CUBIN"] = str(cub)
os.environ["MUSR_NVRTC_OPTS"] = "--ptxas-options=-v"
from paper_1604_02334_b200 import _lib, codegen, workloads  # noqa: E402

ENTRIES = ["musr_chi2_c32", "musr_chi2_c32big", "musr_chi2_f64", "musr_mlh_c32", "musr_mlh_f64",
           "musr_chi2_c32_batch", "musr_mlh_c32_batch"]
CLASSES = {"FP64": ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"), "TMA bulk copy": ("UBLKCP",),
           "mbarrier/SYNCS": ("SYNCS",), "shared load": ("LDS",), "shared store": ("STS",),
           "global/generic load": ("LDG", "LD"), "global store": ("STG", "ST"), "local (spill/stack)": ("LDL", "STL"),
           "MUFU": ("MUFU",), "conversion": ("F2F", "I2F", "F2I"), "atomic": ("ATOMG", "ATOM", "RED", "REDG"),
           "shuffle": ("SHFL",)}

w = workloads.c2(2, 1024)
log = C.create_string_buffer(1 << 20)
size = C.c_size_t()
lib = _lib.load()
assert lib.musr_compile_theory(codegen.lower(w.expr.ast).source.encode(), log, len(log), C.byref(size)) == 0
lines = log.value.decode().splitlines()
props = {}
for i, l in enumerate(lines):
    m = re.search(r"Function properties for (\w+)$", l.strip())
    if m:
        used = lines[i + 2].split(":", 1)[1].strip() if i + 2 < len(lines) and "Used" in lines[i + 2] else ""
        props[m.group(1)] = lines[i + 1].split(".", 1)[1].strip() + ("; " + used if used else "")
print(f"# SASS summary of the product kernels: the library's NVRTC sm_100a compile (musr_compile_theory) of the")
print(f"# C2 / Eq. 6 theory, ptxas -v per entry point and static instruction counts (cuobjdump -sass)")
for e in ENTRIES:
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", e, str(cub)], capture_output=True, text=True).stdout
    ops = Counter(m.split(".")[0] for m in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", sass))
    print(f"\n## {e}: {props.get(e, '?')}")
    print("  total " + str(sum(ops.values())) + "; " + "; ".join(
        f"{k} {sum(ops[x] for x in v)}" for k, v in CLASSES.items()))
