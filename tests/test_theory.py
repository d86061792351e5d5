"""Theory front end: the mirror parser must match the reference DSL
(pkg/src/blk/theory.py:156-406) -- same AST, same postfix code, same errors
and positions -- and the lowering must produce compilable CUDA."""

import ctypes as C

import numpy as np
import pytest

from paper_1604_02334_b200 import codegen, theory
from paper_1604_02334_b200.theory import ParseError, TheoryBinding, TheoryError, parse

K_EQ6 = "p[m[0]] * sg(t, p[m[1]]) * tf(t, p[m[2]] + f[m[4]], 135.538809 * p[m[3]])"

SOURCES = [
    "p[m[0]] * sg(t,p[m[1]]) * tf(t,p[m[2]],f[m[3]])",
    "se(t,p[m[0]])",
    "1.5e3 + 2E-2",
    "2 + 3 * 4", "10 - 4 - 3", "12 / 4 / 3", "2 ^ 3 ^ 2", "2 * 3 ^ 2", "-2 ^ 2", "(2 + 3) * 4",
    "--t", "+-+t", "-t^-2", "t ^ -0.5 ^ 2", ".5 * t", "1. + t", "3e+2 * t",
    K_EQ6,
    "p[m[0]] * stg(t, p[m[1]]) * se(t, p[m[2]]) + p[m[3]] * ge(t, p[m[4]], p[m[5]])",
    "pow(t, p[m[0]]) + sqrt(t) - log(t + 1) / exp(-t) * cos(t) * sin(t)",
    "stg(t, p[m[0]]) / (1 + se(t, p[m[1]]))",
    "p[m[0]]*sg(t,p[m[1]])*tf(t,p[m[2]],f[m[3]]) - se(t, 0.3) ^ 2",
    "p [ m [ 12 ] ] + f[m[0]]",
]

BAD_SOURCES = [
    "sg(t,", "foo(t)", "se(t)", "p[m[1.5]]", "p[0]", "0x10 + t", "t +", "(t", "t)", "p[m[1e1]]",
    "p[k[0]]", "1..2", "t $ 2", "", "exp", "p[m[-1]]", "se(t, 1, 2)", "t t", "p[m[0]", "f[",
    "²", "1.2.3", "2e * t",
]


def test_known_slots_and_positions():
    e = parse("p[m[0]] * sg(t,p[m[1]]) * tf(t,p[m[2]],f[m[3]])")
    assert e.referenced_param_slots == {0, 1, 2}
    assert e.referenced_func_slots == {3}
    with pytest.raises(ParseError) as exc:
        parse("sg(t,")
    assert exc.value.position == 5
    with pytest.raises(ParseError, match="unknown identifier"):
        parse("foo(t)")
    with pytest.raises(ParseError, match="takes 2 arguments"):
        parse("se(t)")
    with pytest.raises(ParseError, match="integer"):
        parse("p[m[1.5]]")


def test_binding_validation():
    b = TheoryBinding(map=(1.0, 2), function_values=(3,))
    assert b.map == (1, 2) and b.function_values == (3.0,)
    with pytest.raises(TheoryError, match="integers"):
        TheoryBinding(map=(1.5,))
    with pytest.raises(TheoryError, match="non-negative"):
        TheoryBinding(map=(-1,))


@pytest.mark.ref
@pytest.mark.parametrize("src", SOURCES)
def test_parse_matches_reference(ref, src):
    mine, theirs = parse(src), ref.theory.parse(src)
    assert mine.bytecode == theirs.bytecode
    assert mine.referenced_param_slots == theirs.referenced_param_slots
    assert mine.referenced_func_slots == theirs.referenced_func_slots
    assert mine.print() == theirs.print()
    assert repr(mine.ast) == repr(theirs.ast).replace("blk.theory.", "")


@pytest.mark.ref
@pytest.mark.parametrize("src", BAD_SOURCES)
def test_parse_errors_match_reference(ref, src):
    with pytest.raises(Exception) as theirs:
        ref.theory.parse(src)
    with pytest.raises(Exception) as mine:
        parse(src)
    assert type(mine.value).__name__ == type(theirs.value).__name__
    assert str(mine.value) == str(theirs.value)
    assert getattr(mine.value, "position", None) == getattr(theirs.value, "position", None)


@pytest.mark.ref
def test_round_trip_property(ref):
    """parse(print(e)) is stable, as the reference's hypothesis test requires."""
    rng = np.random.default_rng(5)
    atoms = ["t", "p[m[0]]", "p[m[1]]", "f[m[2]]", "0.5", "2.0", "1.25e-1"]

    def gen(depth=0):
        if depth >= 3 or rng.random() < 0.4:
            return atoms[rng.integers(len(atoms))]
        kind = rng.integers(4)
        if kind == 0:
            return f"{gen(depth + 1)} {'+-*/'[rng.integers(4)]} {gen(depth + 1)}"
        if kind == 1:
            return f"-{gen(depth + 1)}"
        if kind == 2:
            return f"({gen(depth + 1)})"
        fn = ["se", "sg", "exp", "cos", "sin"][rng.integers(5)]
        return f"{fn}({gen(depth + 1)})" if fn in ("exp", "cos", "sin") else f"{fn}(t, {gen(depth + 1)})"

    for _ in range(300):
        src = gen()
        e = parse(src)
        assert parse(e.print()).bytecode == e.bytecode
        assert e.print() == ref.theory.parse(src).print()


def test_lowering_structure():
    low = codegen.lower(parse(K_EQ6).ast)
    assert low.n_uniform_reg == 4          # A0, sigma, 2*pi*K*B, phase
    assert low.n_rotations == 1            # tf: cos of an affine argument is rotated
    assert low.n_uniform == 4 + 4 * (codegen.ROT_TABLE + 1)
    assert "musr_exp_fast" in low.source and "musr_sincos_fast" in low.source
    assert "musr_cos_fast" in low.source   # the scalar fast body keeps the direct form
    plain = codegen.lower(parse(K_EQ6).ast, rotate=False)
    assert plain.n_rotations == 0 and plain.n_uniform == 4
    assert "musr_theory_exact" in low.source
    # the per-bin body must not touch P/M/F (all slots hoisted)
    body = low.source.split("double musr_theory(")[1].split("}")[0]
    assert "P[" not in body and "F[" not in body
    assert [(e.kind, e.slot) for e in low.events] == [("p", 0), ("p", 1), ("p", 2), ("f", 4),
                                                      ("p", 3)]


def test_lowering_npy_pow_rules():
    src = codegen.lower(parse("t ^ 2 + t ^ 0.5 + t ^ -1 + t ^ 1 + t ^ 0 + t ^ 3 + t ^ p[m[0]] + 2 ^ t").ast).source
    assert "musr_sq(" in src                       # x^2 -> x*x
    assert "__dsqrt_rn(" in src                    # x^0.5 -> sqrt
    assert "__ddiv_rn(1.0," in src                 # x^-1 -> 1/x
    assert "musr_npy_pow_u(" in src                # uniform exponent: numpy's value dispatch
    assert "pow(" in src                           # per-bin exponent: generic pow


def test_literal_folding_and_zero_division_event():
    low = codegen.lower(parse("t + 1 / (2 - 2)").ast)
    assert [e.kind for e in low.events] == ["zdiv"]
    low = codegen.lower(parse("t * (1 / 3)").ast)
    assert "0x1.5555555555555p-2" in low.source   # Python-float 1/3, exactly
    assert low.events == []


@pytest.mark.parametrize("src", SOURCES)
def test_generated_cuda_compiles(src):
    """NVRTC (no device needed) compiles every lowered theory for sm_100a."""
    from paper_1604_02334_b200 import _lib

    lib = _lib.load()
    frag = codegen.lower(parse(src).ast).source
    log = C.create_string_buffer(1 << 16)
    n = C.c_size_t()
    rc = lib.musr_compile_theory(frag.encode(), log, len(log), C.byref(n))
    assert rc == 0, log.value.decode() + lib.musr_global_error().decode()
    assert n.value > 10000
