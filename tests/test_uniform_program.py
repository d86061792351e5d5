"""The host uniform program (codegen._UniformProgram, evaluated per call by the
library's eval_uniform_rows): its instruction stream, restated here as a small
Python interpreter with the library's semantics, must give every U slot exactly
what evaluating the hoisted subtree directly with numpy float64 scalars gives
(the reference's own arithmetic for parameter-only values, theory.py:409-464),
and the library's validation rules must accept it -- for the benchmark theories
and 300 random theories of the GPU fuzz grammar.  No GPU needed."""

import numpy as np
import pytest

from paper_1604_02334_b200 import codegen, workloads
from paper_1604_02334_b200.theory import Binary, Call, Num, SlotRef, Unary, parse

F64 = np.float64
OP = {v: k for k, v in codegen.UOP.items()}


def _npy_pow(x, b):
    if b == 2.0:
        return x * x
    if b == 0.5:
        return np.sqrt(x)
    if b == -1.0:
        return F64(1.0) / x
    if b == 1.0:
        return x
    if b == 0.0:
        return F64(1.0)
    return np.power(x, b)


def _direct(node, P, M, Fv):
    """numpy float64 scalar evaluation of a parameter-only subtree."""
    if isinstance(node, Num):
        return F64(node.value)
    if isinstance(node, SlotRef):
        return F64(P[M[node.slot]]) if node.array == "p" else F64(Fv[M[node.slot]])
    if isinstance(node, Unary):
        return -_direct(node.operand, P, M, Fv)
    if isinstance(node, Binary):
        a, b = _direct(node.left, P, M, Fv), _direct(node.right, P, M, Fv)
        if node.op == "^":
            if isinstance(node.right, Num):
                e = float(node.right.value)
                return _npy_pow(a, e) if e in (2.0, 0.5, -1.0, 1.0, 0.0) else np.power(a, F64(e))
            return _npy_pow(a, b)
        return {"+": np.add, "-": np.subtract, "*": np.multiply, "/": np.divide}[node.op](a, b)
    fn = {"exp": np.exp, "log": np.log, "cos": np.cos, "sin": np.sin, "sqrt": np.sqrt}[node.name]
    return fn(_direct(node.args[0], P, M, Fv))


def _run(code, lits, P, M, Fv, nu_reg, n_rot):
    """The library's eval_uniform_rows + musr_set_uniform_program validation."""
    R, U, rot, nreg = [], [None] * nu_reg, [None] * n_rot, 0
    for k in range(0, len(code), 4):
        op, d, a, b = (OP[code[k]], code[k + 1], code[k + 2], code[k + 3])
        if op == "OUT":
            assert 0 <= d < nu_reg and 0 <= a < nreg
            U[d] = R[a]
            continue
        if op == "ROT":
            assert 0 <= d < n_rot and 0 <= a < nreg
            rot[d] = R[a]
            continue
        assert d == nreg
        nreg += 1
        if op == "LIT":
            v = F64(lits[a])
        elif op in ("P", "F"):
            v = F64(P[M[a]]) if op == "P" else F64(Fv[M[a]])
        else:
            assert 0 <= a < d and (op not in ("ADD", "SUB", "MUL", "DIV", "POWU", "POW") or 0 <= b < d)
            x, y = R[a], (R[b] if b < len(R) else None)
            v = {"NEG": lambda: -x, "ADD": lambda: x + y, "SUB": lambda: x - y, "MUL": lambda: x * y,
                 "DIV": lambda: np.divide(x, y), "SQ": lambda: x * x, "SQRT": lambda: np.sqrt(x),
                 "RCP": lambda: np.divide(F64(1.0), x), "POWU": lambda: _npy_pow(x, y),
                 "POW": lambda: np.power(x, y), "EXP": lambda: np.exp(x), "LOG": lambda: np.log(x),
                 "COS": lambda: np.cos(x), "SIN": lambda: np.sin(x)}[op]()
        R.append(F64(v))
    return U, rot


def _check(src, rng):
    L = codegen.lower(parse(src).ast)
    P = rng.uniform(0.1, 3.0, 8)
    M = list(range(6)) + [6, 7]
    Fv = rng.uniform(-90.0, 90.0, 8)
    with np.errstate(all="ignore"):
        U, rot = _run(L.uniform_code, L.uniform_lits, P, M, Fv, L.n_uniform_reg, L.n_rotations)
        for i, node in enumerate(L.uniform_nodes):
            want = _direct(node, P, M, Fv)
            assert U[i].tobytes() == F64(want).tobytes() or (np.isnan(U[i]) and np.isnan(want)), (src, i)
        for r, w in enumerate(L.rotation_slopes):
            assert rot[r].tobytes() == F64(_direct(w, P, M, Fv)).tobytes(), (src, r)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_benchmark_theories(name):
    w = workloads.WORKLOADS[name](nbins=1024) if name != "C2" else workloads.c2(2, 1024)
    _check(w.expr.source, np.random.default_rng(1))


def test_random_theories():
    import test_gpu_fuzz as fz
    rng = np.random.default_rng(2024)
    for _ in range(300):
        src = fz._term(rng) if rng.random() < 0.7 else fz._term_lp(rng)
        _check(src, rng)
