"""Lower a theory AST to CUDA C++ for the NVRTC JIT (K3).

The generated fragment defines two device functions that the kernel
template in ``csrc/musr_kernel.cuh`` calls:

``musr_uniform(P, M, F, U)``
    evaluated once per histogram tile by one thread; computes every maximal
    parameter-only ("uniform") subexpression into ``U[0..MUSR_NU)``.  This is
    the hoisting of scalar numpy temporaries: in the reference interpreter
    (theory.py:409-464) a subexpression that does not involve ``t`` stays an
    ``np.float64`` scalar and is computed once per call.
``musr_theory(t, U, ok)``
    the per-bin asymmetry A(t) for one bin, in registers, with the branch-free
    fast transcendentals of ``csrc/musr_math.cuh``; clears ``ok`` when an
    argument leaves their fast domain.
``musr_theory_exact(t, U)``
    the same expression with the exact-domain functions; the kernel recomputes
    a thread's bins with it when ``ok`` was cleared (deferred exception check).

Arithmetic contract: every ``+ - * /`` is emitted as a
round-to-nearest intrinsic (``__dadd_rn`` ...), which can never be contracted
into an FMA, in exactly the association order numpy evaluates.  The builtin
shapes are expanded with numpy's operand order (theory.py:62-80):

* ``se(t,l)    = exp((-l) * t)``
* ``ge(t,l,b)  = exp(-(npy_pow(l * t, b)))``
* ``sg(t,s)    = exp(-0.5 * npy_pow(s * t, 2.0))``
* ``stg(t,s)   = 1/3 + ((2/3) * (1 - st2)) * exp(-0.5 * st2)``, ``st2 = npy_pow(s*t, 2.0)``
* ``tf(t,ph,nu)= cos(((2pi * nu) * t) + ((ph * pi) / 180))``

``npy_pow`` follows numpy 2.x ``np.power`` (measured):
with a bin-uniform exponent it short-cuts 2 -> x*x, 0.5 -> sqrt, -1 -> 1/x,
1 -> x, 0 -> 1 and otherwise calls pow; a per-bin exponent always calls pow.

Literal-only ``+ - * /`` subtrees are evaluated by the reference with Python
floats (identical IEEE results, but ``x / 0.0`` raises ZeroDivisionError);
they are folded here with Python floats and a zero divisor is recorded as a
static error event in postfix order, so the objective raises exactly where
the reference would.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from .theory import (
    Binary,
    Call,
    Node,
    Num,
    SlotRef,
    TheoryError,
    TimeVar,
    Unary,
)

__all__ = ["Lowered", "lower", "StaticEvent"]

_TWO_PI = 2.0 * math.pi            # Python float product, == 2.0 * np.pi
_PI = math.pi
_ONE_THIRD = 1.0 / 3.0
_TWO_THIRDS = 2.0 / 3.0


@dataclass(frozen=True)
class StaticEvent:
    """A point in postfix order where the reference interpreter may raise:
    ``kind`` is 'p' / 'f' (slot resolution, theory.py:425-435) or 'zdiv'
    (Python float division by zero of two literals)."""

    kind: str
    slot: int = -1


@dataclass
class Lowered:
    source: str                 # CUDA fragment (musr_uniform + musr_theory)
    n_uniform: int              # MUSR_NU: row length (uniform values + rotation tables)
    uniform_exprs: List[str]    # readable form of each U slot (docs / debugging)
    events: List[StaticEvent]   # postfix-ordered raise points
    max_p_slot: int             # largest k in p[m[k]] (-1 if none)
    max_f_slot: int             # largest k in f[m[k]] (-1 if none)
    per_bin: bool               # does A depend on t at all
    n_uniform_reg: int = 1      # MUSR_NU_REG: leading row entries kept in registers
    n_rotations: int = 0        # MUSR_NROT: rotated cos/sin arguments
    # the uniform row as a host program (musr_set_uniform_program): int32
    # quadruples (op, dst, a, b) over a register file, and its literals
    uniform_code: List[int] = field(default_factory=list)
    uniform_lits: List[float] = field(default_factory=list)
    uniform_nodes: List[Node] = field(default_factory=list)   # the hoisted subtrees, U order
    rotation_slopes: List[Node] = field(default_factory=list)  # W of each rotation table


# -- static events + literal folding on the user AST --------------------------

class _ZeroDiv:
    """Marker for a literal subtree whose evaluation raises."""


def _events_and_fold(node: Node, events: List[StaticEvent]):
    """Return (folded_node, pyfloat_value_or_None).  ``pyfloat`` is the Python
    float the reference would hold for a literal-only subtree."""
    if isinstance(node, Num):
        return node, float(node.value)
    if isinstance(node, TimeVar):
        return node, None
    if isinstance(node, SlotRef):
        events.append(StaticEvent(node.array, node.slot))
        return node, None
    if isinstance(node, Unary):
        inner, val = _events_and_fold(node.operand, events)
        if isinstance(val, float):
            return Num(-val), -val
        return Unary("-", inner), None
    if isinstance(node, Binary):
        left, lv = _events_and_fold(node.left, events)
        right, rv = _events_and_fold(node.right, events)
        if node.op != "^" and isinstance(lv, float) and isinstance(rv, float):
            if node.op == "+":
                v = lv + rv
            elif node.op == "-":
                v = lv - rv
            elif node.op == "*":
                v = lv * rv
            else:
                if rv == 0.0:
                    events.append(StaticEvent("zdiv"))
                    return Binary(node.op, left, right), _ZeroDiv
                v = lv / rv
            return Num(v), v
        return Binary(node.op, left, right), None
    if isinstance(node, Call):
        args = tuple(_events_and_fold(a, events)[0] for a in node.args)
        return Call(node.name, args), None
    raise TheoryError(f"unknown node {node!r}")


# -- builtin expansion to primitives --------------------------------------------

def _exp(x: Node) -> Node:
    return Call("exp", (x,))


def _desugar(node: Node) -> Node:
    if isinstance(node, (Num, TimeVar, SlotRef)):
        return node
    if isinstance(node, Unary):
        return Unary("-", _desugar(node.operand))
    if isinstance(node, Binary):
        return Binary(node.op, _desugar(node.left), _desugar(node.right))
    if not isinstance(node, Call):
        raise TheoryError(f"unknown node {node!r}")
    a = tuple(_desugar(x) for x in node.args)
    name = node.name
    if name in ("exp", "log", "cos", "sin", "sqrt"):
        return Call(name, a)
    if name == "pow":
        return Binary("^", a[0], a[1])
    if name == "se":
        t, lam = a
        return _exp(Binary("*", Unary("-", lam), t))
    if name == "ge":
        t, lam, beta = a
        return _exp(Unary("-", Binary("^", Binary("*", lam, t), beta)))
    if name == "sg":
        t, sigma = a
        return _exp(Binary("*", Num(-0.5), Binary("^", Binary("*", sigma, t), Num(2.0))))
    if name == "stg":
        t, sigma = a
        st2 = Binary("^", Binary("*", sigma, t), Num(2.0))
        damp = _exp(Binary("*", Num(-0.5), st2))
        return Binary(
            "+",
            Num(_ONE_THIRD),
            Binary("*", Binary("*", Num(_TWO_THIRDS), Binary("-", Num(1.0), st2)), damp),
        )
    if name == "tf":
        t, phi, nu = a
        omega_t = Binary("*", Binary("*", Num(_TWO_PI), nu), t)
        phase = Binary("/", Binary("*", phi, Num(_PI)), Num(180.0))
        return Call("cos", (Binary("+", omega_t, phase),))
    raise TheoryError(f"unknown function {name!r}")


# -- emission ---------------------------------------------------------------------

def _lit(v: float) -> str:
    """Exact C++ double literal."""
    if math.isnan(v):
        return "__longlong_as_double(0x7ff8000000000000LL)"
    if math.isinf(v):
        return "__longlong_as_double(0x7ff0000000000000LL)" if v > 0 else \
            "__longlong_as_double(0xfff0000000000000LL)"
    if v == 0.0:
        return "(-0.0)" if math.copysign(1.0, v) < 0 else "0.0"
    return f"({v.hex()})"


def _depends_on_t(node: Node, memo: Dict[Node, bool]) -> bool:
    if node in memo:
        return memo[node]
    if isinstance(node, TimeVar):
        r = True
    elif isinstance(node, (Num, SlotRef)):
        r = False
    elif isinstance(node, Unary):
        r = _depends_on_t(node.operand, memo)
    elif isinstance(node, Binary):
        r = _depends_on_t(node.left, memo) or _depends_on_t(node.right, memo)
    else:
        r = any(_depends_on_t(x, memo) for x in node.args)
    memo[node] = r
    return r


_ARITH = {"+": "__dadd_rn", "-": "__dsub_rn", "*": "__dmul_rn", "/": "__ddiv_rn"}
_FUNC_EXACT = {             # uniform prologue and the rare exact fallback
    "exp": "musr_exp",      # csrc/musr_math.cuh: <= 1 ulp, libdevice beyond |x| > 708
    "log": "log",
    "cos": "musr_cos",      # abs. error <= 2.5e-16 for |x| < 2^20, libdevice beyond
    "sin": "musr_sin",
    "sqrt": "__dsqrt_rn",
}
_FUNC_FAST = {              # hot loop: branch-free, clear `ok` outside the fast domain
    "exp": "musr_exp_fast",
    "cos": "musr_cos_fast",
    "sin": "musr_sin_fast",
}


class _Emitter:
    """SSA emitter with structural CSE (identical subtrees computed once,
    which is bit-neutral)."""

    def __init__(self, leaf, fast: bool = False):
        self.lines: List[str] = []
        self.names: Dict[Node, str] = {}
        self.leaf = leaf          # callback for TimeVar/SlotRef/hoisted nodes
        self.uniform_of = None    # callback: is the node bin-uniform?
        self.fast = fast          # emit *_fast(x, ok) variants

    def value(self, node: Node) -> str:
        if isinstance(node, Num):
            return _lit(float(node.value))
        direct = self.leaf(node)
        if direct is not None:
            return direct
        if node in self.names:
            return self.names[node]
        expr = self._expr(node)
        name = f"v{len(self.names)}"
        self.lines.append(f"  const double {name} = {expr};")
        self.names[node] = name
        return name

    def _expr(self, node: Node) -> str:
        if isinstance(node, Unary):
            return f"(-{self.value(node.operand)})"
        if isinstance(node, Binary):
            if node.op == "^":
                return self._pow(node)
            return f"{_ARITH[node.op]}({self.value(node.left)}, {self.value(node.right)})"
        if isinstance(node, Call):
            arg = self.value(node.args[0])
            if self.fast and node.name in _FUNC_FAST:
                return f"{_FUNC_FAST[node.name]}({arg}, ok)"
            return f"{_FUNC_EXACT[node.name]}({arg})"
        raise TheoryError(f"cannot emit {node!r}")

    def _pow(self, node: Binary) -> str:
        base = self.value(node.left)
        ex = node.right
        if isinstance(ex, Num):
            e = float(ex.value)
            if e == 2.0:
                return f"musr_sq({base})"
            if e == 0.5:
                return f"__dsqrt_rn({base})"
            if e == -1.0:
                return f"__ddiv_rn(1.0, {base})"
            if e == 1.0:
                return base
            if e == 0.0:
                return "1.0"
            return f"pow({base}, {_lit(e)})"
        if self.uniform_of(ex):
            return f"musr_npy_pow_u({base}, {self.value(ex)})"
        return f"pow({base}, {self.value(ex)})"


class _VecEmitter:
    """Per-bin body vectorised over a thread's MUSR_PT consecutive bins.

    Per-bin values are arrays ``vN[MUSR_PT]``; bin-uniform ones are scalars.
    exp and bin-uniform-exponent pow are *anchored* on the run's first bin
    (csrc/musr_math.cuh: musr_exp_anchored / musr_pow_anchored): one full
    evaluation per run plus a short series per further bin, with the error
    bounded per bin (no accumulation).

    cos/sin of an argument affine in t with uniform coefficients,
    ``a(t) = W*t (+/- Phi)`` -- the ``tf`` precession -- are *rotated*: the
    argument a_j of every bin is computed exactly as the reference does, the
    run's first bin gets one full sincos (c0, s0), and bin j uses the
    per-dataset table (D_j = W*(j*dt), cos D_j, sin D_j) built with the
    uniform row:  cos(a_j) = c0*X_j - s0*Y_j,  sin(a_j) = s0*X_j + c0*Y_j,
    with X_j = cos D_j - e_j*sin D_j, Y_j = sin D_j + e_j*cos D_j and
    e_j = (a_j - a_0) - D_j (the rotation of (c0, s0) by D_j + e_j to first
    order; |e_j| ~ ulp(a), so the dropped e_j^2 term is < 2^-62).  Per bin 6
    FP64 operations instead of a reduction and a degree-8 polynomial; the error
    stays bounded per bin (every run restarts from an evaluated anchor).
    Any argument outside a fast form's window clears ``ok``.
    """

    def __init__(self, scalar_leaf, uniform_of, rotations=None):
        self.lines: List[str] = []
        self.names: Dict[Node, str] = {}
        self.scalar_leaf = scalar_leaf   # uniform node -> C expression (U[k] / literal)
        self.uniform_of = uniform_of
        self.n = 0
        self.rotations = rotations       # {arg node: table index}, None = no rotation

    def _fresh(self) -> str:
        self.n += 1
        return f"w{self.n}"

    def ref(self, node: Node, j: str) -> str:
        """C expression of `node` at bin index expression `j`."""
        if isinstance(node, Num):
            return _lit(float(node.value))
        if isinstance(node, TimeVar):
            return f"t[{j}]"
        if self.uniform_of(node):
            return self.scalar_leaf(node)
        return f"{self.vec(node)}[{j}]"

    def _loop(self, name: str, body: str, first: int = 0) -> None:
        self.lines.append(f"  #pragma unroll")
        self.lines.append(f"  for (int j = {first}; j < MUSR_PT; ++j) {name}[j] = {body};")

    def vec(self, node: Node) -> str:
        if node in self.names:
            return self.names[node]
        name = self._fresh()
        self.lines.append(f"  double {name}[MUSR_PT];")
        if isinstance(node, Unary):
            self._loop(name, f"(-{self.ref(node.operand, 'j')})")
        elif isinstance(node, Binary) and node.op != "^":
            self._loop(name, f"{_ARITH[node.op]}({self.ref(node.left, 'j')}, {self.ref(node.right, 'j')})")
        elif isinstance(node, Binary):
            self._pow(name, node)
        elif isinstance(node, Call):
            self._call(name, node)
        else:
            raise TheoryError(f"cannot vectorise {node!r}")
        self.names[node] = name
        return name

    def _call(self, name: str, node: Call) -> None:
        arg = node.args[0]
        if node.name == "exp":
            if self.uniform_of(arg):  # cannot happen: uniform calls are hoisted
                raise TheoryError("uniform exp reached the vector emitter")
            # exp(c * y) with c = +-2^k (the -0.5 of sg / stg): anchored on y with the
            # series coefficients scaled by c^k -- bit-identical, no per-bin multiply
            scaled = _pow2_scaled(arg, self.uniform_of)
            c, y = scaled if scaled is not None else (1.0, arg)
            yv = "t" if isinstance(y, TimeVar) else self.vec(y)
            x0 = f"{yv}[0]" if c == 1.0 else f"__dmul_rn({_lit(c)}, {yv}[0])"
            k = int(math.log2(abs(c)))
            b = [c ** 4 * float.fromhex("0x1.5555555555555p-5"),
                 c ** 3 * float.fromhex("0x1.5555555555555p-3"), c * c * 0.5, c]
            hi10, hi13 = (1023 - 10 - k) << 20, (1023 - 13 - k) << 20
            dd, hm = self._fresh(), self._fresh()
            self.lines.append(f"  {name}[0] = musr_exp_fast({x0}, ok);")
            self.lines.append(f"  double {dd}[MUSR_PT]; int {hm} = 0;")
            self.lines.append(f"  #pragma unroll")
            self.lines.append(f"  for (int j = 1; j < MUSR_PT; ++j) {{ {dd}[j] = __dsub_rn({yv}[j], {yv}[0]); "
                              f"{hm} = max({hm}, musr_hiabs({dd}[j])); }}")
            self.lines.append(f"  ok = ok && {hm} < {hi10:#x};  // |d| < 2^-10 (d = c * dy)")
            self.lines.append(f"  if (MUSR_EXP_DEG3 && {hm} < {hi13:#x}) {{  // |d| < 2^-13: degree 3")
            self._loop(name, f"musr_exp_series3({dd}[j], {name}[0], {_lit(b[1])}, {_lit(b[2])}, {_lit(b[3])})",
                       first=1)
            self.lines.append("  } else {")
            self._loop(name, f"musr_exp_series4({dd}[j], {name}[0], {', '.join(_lit(x) for x in b)})", first=1)
            self.lines.append("  }")
        elif node.name in ("cos", "sin") and self.rotations is not None and arg in self.rotations:
            self._rotated(name, node.name, arg, self.rotations[arg])
        elif node.name in ("cos", "sin"):
            self._loop(name, f"musr_{node.name}_fast({self.ref(arg, 'j')}, ok)")
        elif node.name == "sqrt":
            self._loop(name, f"__dsqrt_rn({self.ref(arg, 'j')})")
        else:
            self._loop(name, f"{_FUNC_EXACT[node.name]}({self.ref(arg, 'j')})")

    def _rotated(self, name: str, fn: str, arg: Node, r: int) -> None:
        a = self.vec(arg)
        tab = f"(R + MUSR_NU_REG + 4 * MUSR_PT * {r})"
        # cos(a0 + D + e) = c0*X - s0*Y, sin(a0 + D + e) = s0*X + c0*Y with
        # X = cos D - e*sin D, Y = sin D + e*cos D (first order in e; e^2 < 2^-62)
        out = ("__fma_rn(c0_, X_, -__dmul_rn(s0_, Y_))" if fn == "cos"
               else "__fma_rn(s0_, X_, __dmul_rn(c0_, Y_))")
        self.lines.append(f"  {{ double s0_, c0_;")
        self.lines.append(f"    musr_sincos_fast({a}[0], &s0_, &c0_, ok);")
        self.lines.append(f"    {name}[0] = {'c0_' if fn == 'cos' else 's0_'};")
        self.lines.append(f"    #pragma unroll")
        self.lines.append(f"    for (int j = 1; j < MUSR_PT; ++j) {{")
        self.lines.append(f"      const double* tb_ = {tab} + 4 * j;  // (D_j, cos D_j | sin D_j, -)")
        self.lines.append(f"      const double2 dc_ = *reinterpret_cast<const double2*>(tb_);")
        self.lines.append(f"      const double sj_ = tb_[2];")
        self.lines.append(f"      const double e_ = __dsub_rn(__dsub_rn({a}[j], {a}[0]), dc_.x);")
        self.lines.append(f"      ok = ok && musr_abs_below(e_, 0x3e000000);  // |e| < 2^-31")
        self.lines.append(f"      const double X_ = __fma_rn(-sj_, e_, dc_.y);")
        self.lines.append(f"      const double Y_ = __fma_rn(dc_.y, e_, sj_);")
        self.lines.append(f"      {name}[j] = {out};")
        self.lines.append(f"    }} }}")

    def _pow(self, name: str, node: Binary) -> None:
        base, ex = node.left, node.right
        if not self.uniform_of(base) and not isinstance(base, TimeVar):
            self.vec(base)  # materialise before any branch so every path can use it
        bj = lambda: self.ref(base, "j")
        if isinstance(ex, Num):
            e = float(ex.value)
            special = {2.0: "musr_sq({b})", 0.5: "__dsqrt_rn({b})", -1.0: "__ddiv_rn(1.0, {b})",
                       1.0: "{b}", 0.0: "1.0"}
            if e in special:
                self._loop(name, special[e].format(b=bj()))
                return
            self._anchored_pow(name, base, _lit(e))
            return
        if self.uniform_of(ex):
            b = self.scalar_leaf(ex)
            self.lines.append(f"  if ({b} == 2.0 || {b} == 0.5 || {b} == -1.0 || {b} == 1.0 || {b} == 0.0) {{")
            self._loop(name, f"musr_npy_pow_u({bj()}, {b})")
            self.lines.append("  } else {")
            self._anchored_pow(name, base, b)
            self.lines.append("  }")
            return
        self._loop(name, f"pow({bj()}, {self.ref(ex, 'j')})")

    def _anchored_pow(self, name: str, base: Node, b: str) -> None:
        x0 = self.ref(base, "0")
        # anchor: exp(b * log x0) in extended precision (musr_pow_fast, <= 2 ulp);
        # outside its domain `ok` drops and the thread's bins are redone exactly
        self.lines.append(f"  {{ const double p0_ = MUSR_POW_ANCHOR({x0}, {b}, ok);")
        self.lines.append(f"    const MusrPowAnchor an_ = musr_pow_anchor({x0}, p0_, {b});")
        self.lines.append(f"    {name}[0] = p0_;")
        self.lines.append(f"    #pragma unroll")
        self.lines.append(f"    for (int j = 1; j < MUSR_PT; ++j) {name}[j] = musr_pow_anchored({self.ref(base, 'j')}, an_, ok); }}")


def _pow2_scaled(arg: Node, uniform) -> Optional[Tuple[float, Node]]:
    """(c, y) when ``arg`` is ``c * y`` or ``y * c`` with c a literal +-2^k
    (|k| <= 8, so the scaled series coefficients stay normal) and y per-bin."""
    if not (isinstance(arg, Binary) and arg.op == "*"):
        return None
    for lit, y in ((arg.left, arg.right), (arg.right, arg.left)):
        if isinstance(lit, Num) and not uniform(y):
            c = float(lit.value)
            if c != 0.0 and math.isfinite(c):
                m, e = math.frexp(abs(c))
                if m == 0.5 and -8 <= e - 1 <= 8:
                    return c, y
    return None


# Opcodes of the host uniform program (csrc/musr_b200.cu: eval_uniform_row).  Each
# mirrors the device prologue's operation (_Emitter) with IEEE double arithmetic;
# exp / log / cos / sin / pow are the host libm's, as numpy's float64 scalars use.
UOP = {"LIT": 0, "P": 1, "F": 2, "NEG": 3, "ADD": 4, "SUB": 5, "MUL": 6, "DIV": 7, "SQ": 8,
       "SQRT": 9, "RCP": 10, "POWU": 11, "POW": 12, "EXP": 13, "LOG": 14, "COS": 15, "SIN": 16,
       "OUT": 17, "ROT": 18}
_UOP_BIN = {"+": "ADD", "-": "SUB", "*": "MUL", "/": "DIV"}
_UOP_CALL = {"exp": "EXP", "log": "LOG", "cos": "COS", "sin": "SIN", "sqrt": "SQRT"}


class _UniformProgram:
    """The uniform prologue (U slots and rotation-table slopes) as a register
    program the host library evaluates per call; same CSE and operation choice
    as the device emitter, so arithmetic-only rows are bit-identical to it."""

    def __init__(self):
        self.code: List[int] = []
        self.lits: List[float] = []
        self.regs: Dict[Node, int] = {}
        self.n = 0

    def _emit(self, op: str, a: int = 0, b: int = 0) -> int:
        dst = self.n
        self.n += 1
        self.code += [UOP[op], dst, a, b]
        return dst

    def lit(self, v: float) -> int:
        self.lits.append(float(v))
        return self._emit("LIT", len(self.lits) - 1)

    def reg(self, node: Node) -> int:
        if isinstance(node, Num):
            return self.lit(float(node.value))
        if node in self.regs:
            return self.regs[node]
        if isinstance(node, SlotRef):
            r = self._emit("P" if node.array == "p" else "F", node.slot)
        elif isinstance(node, Unary):
            r = self._emit("NEG", self.reg(node.operand))
        elif isinstance(node, Binary) and node.op != "^":
            r = self._emit(_UOP_BIN[node.op], self.reg(node.left), self.reg(node.right))
        elif isinstance(node, Binary):
            base, ex = self.reg(node.left), node.right
            if isinstance(ex, Num):
                e = float(ex.value)
                if e == 2.0:
                    r = self._emit("SQ", base)
                elif e == 0.5:
                    r = self._emit("SQRT", base)
                elif e == -1.0:
                    r = self._emit("RCP", base)
                elif e == 1.0:
                    r = base
                elif e == 0.0:
                    r = self.lit(1.0)
                else:
                    r = self._emit("POW", base, self.lit(e))
            else:
                r = self._emit("POWU", base, self.reg(ex))
        elif isinstance(node, Call):
            r = self._emit(_UOP_CALL[node.name], self.reg(node.args[0]))
        else:
            raise TheoryError(f"internal: {node!r} in a uniform subtree")
        self.regs[node] = r
        return r

    def out(self, slot: int, node: Node) -> None:
        self.code += [UOP["OUT"], slot, self.reg(node), 0]

    def rot(self, r: int, slope: Node) -> None:
        self.code += [UOP["ROT"], r, self.reg(slope), 0]


ROT_TABLE = 15  # bins per run a rotation table covers (MUSR_PT <= ROT_TABLE + 1)


def _affine_slope(arg: Node, uniform) -> Optional[Node]:
    """W when ``arg`` is ``W*t``, ``t*W``, ``W*t +/- Phi`` or ``Phi + W*t`` with W
    and Phi bin-uniform, else None."""
    def slope(x):
        if isinstance(x, Binary) and x.op == "*":
            if isinstance(x.right, TimeVar) and uniform(x.left):
                return x.left
            if isinstance(x.left, TimeVar) and uniform(x.right):
                return x.right
        return None

    w = slope(arg)
    if w is not None:
        return w
    if isinstance(arg, Binary) and arg.op in ("+", "-"):
        w = slope(arg.left)
        if w is not None and uniform(arg.right):
            return w
        if arg.op == "+" and uniform(arg.left):
            return slope(arg.right)
    return None


def lower(ast: Node, rotate: bool = True) -> Lowered:
    events: List[StaticEvent] = []
    folded, pyval = _events_and_fold(ast, events)
    prim = _desugar(folded)

    memo: Dict[Node, bool] = {}
    per_bin = _depends_on_t(prim, memo)

    def uniform(n: Node) -> bool:
        return not _depends_on_t(n, memo)

    # 1) collect maximal uniform, non-literal subtrees (hoisted to U)
    hoisted: Dict[Node, int] = {}
    order: List[Node] = []

    def collect(n: Node) -> None:
        if isinstance(n, Num):
            return
        if uniform(n):
            if n not in hoisted:
                hoisted[n] = len(order)
                order.append(n)
            return
        if isinstance(n, Unary):
            collect(n.operand)
        elif isinstance(n, Binary):
            collect(n.left)
            collect(n.right)
        elif isinstance(n, Call):
            for x in n.args:
                collect(x)

    collect(prim)
    if not per_bin and not isinstance(prim, Num) and not order:
        order.append(prim)
        hoisted[prim] = 0

    # cos/sin of affine arguments get a per-dataset rotation table
    rotations: Dict[Node, int] = {}
    slopes: List[Node] = []

    def find_rot(n: Node) -> None:
        if isinstance(n, Call) and n.name in ("cos", "sin") and not uniform(n):
            a = n.args[0]
            w = _affine_slope(a, uniform)
            if w is not None and a not in rotations:
                rotations[a] = len(slopes)
                slopes.append(w)
        for c in (n.operand,) if isinstance(n, Unary) else (n.left, n.right) \
                if isinstance(n, Binary) else n.args if isinstance(n, Call) else ():
            find_rot(c)

    if rotate and per_bin:
        find_rot(prim)

    # 2) uniform prologue: slot loads through the per-histogram map row
    def uleaf(n: Node) -> Optional[str]:
        if isinstance(n, SlotRef):
            arr = "P" if n.array == "p" else "F"
            return f"{arr}[M[{n.slot}]]"
        if isinstance(n, TimeVar):
            raise TheoryError("internal: t inside a uniform subtree")
        return None

    ue = _Emitter(uleaf)
    ue.uniform_of = lambda n: True
    u_lines: List[str] = []
    for i, n in enumerate(order):
        ue.lines = []
        val = ue.value(n)
        u_lines.extend(ue.lines)
        u_lines.append(f"  U[{i}] = {val};")
    nu_reg = max(len(order), 1)
    uprog = _UniformProgram()
    for i, n in enumerate(order):
        uprog.out(i, n)
    if not order:
        uprog.code += [UOP["OUT"], 0, uprog.lit(0.0), 0]
    for r, w in enumerate(slopes):
        uprog.rot(r, w)
    rot_lines: List[str] = []
    for r, w in enumerate(slopes):   # rotation table entry j: D_j = W*(j*dt), cos D_j, sin D_j
        wv = _lit(float(w.value)) if isinstance(w, Num) else f"U[{hoisted[w]}]"
        base = f"(MUSR_NU_REG + 4 * MUSR_PT * {r})"
        rot_lines.append(f"  {{ const double d_ = __dmul_rn({wv}, __dmul_rn((double)j, dt));")
        rot_lines.append("    double s_, c_; bool ok_ = true;")
        rot_lines.append("    musr_sincos_fast(d_, &s_, &c_, ok_);")
        rot_lines.append("    if (!ok_) { c_ = musr_cos(d_); s_ = musr_sin(d_); }")
        rot_lines.append(f"    U[{base} + 4 * j] = d_; U[{base} + 4 * j + 1] = c_; "
                         f"U[{base} + 4 * j + 2] = s_; U[{base} + 4 * j + 3] = 0.0; }}")

    # 3) per-bin body: a branch-free fast variant that clears `ok` when an
    #    argument leaves the fast domain, and the exact variant the kernel
    #    falls back to (reading the uniform row from memory, so the hot loop's
    #    registers are never forced to local memory).
    def bleaf(n: Node) -> Optional[str]:
        if isinstance(n, TimeVar):
            return "t"
        if n in hoisted:
            return f"U[{hoisted[n]}]"
        return None

    bodies = {}
    for fast in (True, False):
        be = _Emitter(bleaf, fast=fast)
        be.uniform_of = uniform
        result = be.value(prim)
        bodies[fast] = (be.lines, result)

    nu = len(order)
    # rotation entries are 32-byte aligned (one 16-byte and one 8-byte load):
    # pad the register part to an even count, and the row (+ N0, Nbkg) stays even
    if slopes and nu_reg % 2:
        nu_reg += 1
    # rotation tables hold MUSR_PT entries (the row length follows the tile
    # configuration the kernel is compiled for); n_row is the MUSR_PT = 16 maximum
    n_row = nu_reg + 4 * (ROT_TABLE + 1) * len(slopes)
    src: List[str] = []
    src.append(f"#define MUSR_NU_REG {nu_reg}")
    src.append(f"#define MUSR_NROT {len(slopes)}")
    src.append("#define MUSR_NU (MUSR_NU_REG + 4 * MUSR_PT * MUSR_NROT)")
    if slopes:
        src.append(f"#if MUSR_PT > {ROT_TABLE + 1}")
        src.append("#error rotation tables cover at most 16 bins per run")
        src.append("#endif")
    src.append("__device__ __forceinline__ void musr_uniform(const double* __restrict__ P, "
               "const int* __restrict__ M, const double* __restrict__ F, "
               "double* __restrict__ U) {")
    src.append("  (void)P; (void)M; (void)F;")
    src.extend(u_lines)
    if nu == 0:
        src.append("  U[0] = 0.0;")
    src.append("}")
    # rotation-table entry j (1 <= j < MUSR_PT) of a row whose uniform part U is set
    src.append("__device__ __forceinline__ void musr_rot_entry(double* __restrict__ U, "
               "const double dt, const int j) {")
    src.append("  (void)U; (void)dt; (void)j;")
    src.extend(rot_lines)
    src.append("}")
    src.append("__device__ __forceinline__ double musr_theory(const double t, "
               "const double* __restrict__ U, bool& ok) {")
    src.append("  (void)t; (void)U; (void)ok;")
    src.extend(bodies[True][0])
    src.append(f"  return {bodies[True][1]};")
    src.append("}")
    # vectorised per-thread body (anchored transcendentals)
    ve = _VecEmitter(lambda n: _lit(float(n.value)) if isinstance(n, Num) else f"U[{hoisted[n]}]",
                     uniform, rotations if rotate else None)
    if per_bin:
        vres = ve.vec(prim) if not isinstance(prim, TimeVar) else None
    src.append("__device__ __forceinline__ void musr_theory_vec(const double (&t)[MUSR_PT], "
               "const double* __restrict__ U, const double* __restrict__ R, "
               "double (&A)[MUSR_PT], bool& ok) {")
    src.append("  (void)t; (void)U; (void)R; (void)ok;")
    if not per_bin:
        val = _lit(float(prim.value)) if isinstance(prim, Num) else f"U[{hoisted[prim]}]"
        src.append("  #pragma unroll")
        src.append(f"  for (int j = 0; j < MUSR_PT; ++j) A[j] = {val};")
    elif isinstance(prim, TimeVar):
        src.append("  #pragma unroll")
        src.append("  for (int j = 0; j < MUSR_PT; ++j) A[j] = t[j];")
    else:
        src.extend(ve.lines)
        src.append("  #pragma unroll")
        src.append(f"  for (int j = 0; j < MUSR_PT; ++j) A[j] = {vres}[j];")
    src.append("}")
    src.append("__device__ __noinline__ double musr_theory_exact(const double t, "
               "const double* __restrict__ U) {")
    src.append("  (void)t; (void)U;")
    src.extend(bodies[False][0])
    src.append(f"  return {bodies[False][1]};")
    src.append("}")

    p_slots = [e.slot for e in events if e.kind == "p"]
    f_slots = [e.slot for e in events if e.kind == "f"]
    return Lowered(
        source="\n".join(src) + "\n",
        n_uniform=n_row,
        n_uniform_reg=nu_reg,
        n_rotations=len(slopes),
        uniform_exprs=[_readable(n) for n in order],
        events=events,
        max_p_slot=max(p_slots, default=-1),
        max_f_slot=max(f_slots, default=-1),
        per_bin=per_bin,
        uniform_code=uprog.code,
        uniform_lits=uprog.lits,
        uniform_nodes=list(order),
        rotation_slopes=list(slopes),
    )


def _readable(n: Node) -> str:
    if isinstance(n, Num):
        return repr(n.value)
    if isinstance(n, TimeVar):
        return "t"
    if isinstance(n, SlotRef):
        return f"{n.array}[m[{n.slot}]]"
    if isinstance(n, Unary):
        return f"(-{_readable(n.operand)})"
    if isinstance(n, Binary):
        return f"({_readable(n.left)} {n.op} {_readable(n.right)})"
    return f"{n.name}({', '.join(_readable(a) for a in n.args)})"
