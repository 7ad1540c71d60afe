"""Host-side logic and the C-ABI boundary (CPU, no GPU needed)."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from paper_1709_03187_b200 import (CONFIGS, Instance, InvalidArgument, Mode, PacoError, ParseError, RunConfig,
                                   cycle_length, emit_tsplib, euc2d, grid_instance, is_permutation_of_n, load_optima,
                                   make_config_instance, mode_from_name, mode_name, parse_tsplib, tour_length)
from paper_1709_03187_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ instances (instance.hpp)

def test_euc2d_kats():
    """test_instance.cpp:136-145"""
    inst = Instance.from_coords("grid", [(0, 0), (3, 4), (1, 1), (0.5, 0), (10, 0)])
    assert [inst.dist(0, j) for j in range(5)] == [0, 5, 1, 1, 10]
    assert inst.dist(1, 0) == inst.dist(0, 1)
    assert euc2d(0, 0, 3, 4) == 5


def test_tour_length_and_validation():
    """test_instance.cpp:171-200"""
    tri = Instance.from_coords("tri", [(0, 0), (3, 0), (3, 4)])
    assert tour_length(tri, [0, 1, 2]) == 12
    with pytest.raises(ValueError):
        tour_length(tri, [0, 1, 1])
    with pytest.raises(ValueError):
        tour_length(tri, [0, 1])
    rng = np.random.default_rng(23)
    inst = Instance("r", rng.random(7) * 1000, rng.random(7) * 1000)
    order = rng.permutation(7)
    base = tour_length(inst, order)
    assert tour_length(inst, np.roll(order, 3)) == base
    assert tour_length(inst, order[::-1]) == base
    assert is_permutation_of_n(7, order) and not is_permutation_of_n(7, [0] * 7)


def test_instance_validation():
    with pytest.raises(ValueError):
        Instance.from_coords("two", [(0, 0), (1, 1)])
    with pytest.raises(ValueError):
        Instance("nan", np.array([0.0, 1.0, np.nan]), np.zeros(3))
    with pytest.raises(ValueError):
        Instance.from_coords("opt", [(0, 0), (1, 0), (0, 1)], optimum=0)


def test_tsplib_round_trip_and_errors():
    """instance.hpp:164-261: emit -> parse is exact; errors carry line numbers."""
    inst = make_config_instance("C3", n=50)
    back = parse_tsplib(emit_tsplib(inst))
    assert np.array_equal(back.xs, inst.xs) and np.array_equal(back.ys, inst.ys) and back.name == inst.name
    frac = Instance.from_coords("f", [(0.1, 1e-3), (123456.789, 2.5), (1 / 3, 7.0)])
    back = parse_tsplib(emit_tsplib(frac))
    assert np.array_equal(back.xs, frac.xs)
    bad = [
        ("NAME: x\nNODE_COORD_SECTION\n", 2, "before DIMENSION"),
        ("DIMENSION: 3\nNODE_COORD_SECTION\n", 2, "EDGE_WEIGHT_TYPE"),
        ("DIMENSION: 3\nEDGE_WEIGHT_TYPE: GEO\n", 2, "unsupported"),
        ("DIMENSION: x\n", 1, "non-numeric"),
        ("DIMENSION: 2\n", 1, "at least 3"),
        ("garbage line\n", 1, "malformed"),
        ("DIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1\n", 5, "expected"),
        ("DIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0 9\n", 4, "trailing"),
        ("DIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\nEOF\n", 6, "DIMENSION is 3"),
        ("DIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\n", 2, "missing NODE_COORD_SECTION"),
    ]
    for text, line, msg in bad:
        with pytest.raises(ParseError) as ei:
            parse_tsplib(text)
        assert ei.value.line == line and msg in str(ei.value), (text, str(ei.value))


def test_optima_and_grid442():
    """data/README.md:7-10: 26x17 grid at spacing 10 has optimum 4420 (regenerated, not copied)."""
    g = grid_instance(26, 17, 10.0, "grid442")
    assert g.n == 442 and g.optimum == 4420
    order = [r * 26 + (c if r % 2 == 0 else 25 - c) for r in range(17) for c in range(26)]
    assert cycle_length(g, order) > 4420  # boustrophedon over 17 rows needs a long closing edge
    opt = load_optima("# c\ngrid442 4420\npcb442 50778\n")
    assert opt == {"grid442": 4420, "pcb442": 50778}
    with pytest.raises(ParseError):
        load_optima("x -1\n")


def test_reference_test_instance_generator():
    """tests/refgen.py reproduces oracles.hpp:123-131 (std::mt19937_64 + uniform_real_distribution,
    libstdc++): values printed by a g++ 13 build of the same calls."""
    from refgen import MT19937_64, random_instance
    g = MT19937_64()
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042  # [rand.predef]: 10000th output of the default-seeded engine
    g3 = MT19937_64(3)
    assert (g3(), g3()) == (10307413207671831467, 3611203882987592167)
    inst = random_instance(MT19937_64(3), 3)
    assert inst.xs.tolist() == [195.76375476116183, 346.36890921172545, 361.30268965844164]
    assert inst.ys.tolist() == [558.76598962317905, 590.24127156131578, 559.79563654389858]


def test_config_instances_shapes_and_determinism():
    for name, spec in CONFIGS.items():
        small = make_config_instance(name, n=2000)
        again = make_config_instance(name, n=2000)
        assert small.sha256() == again.sha256()
        assert small.xs.min() >= 0 and small.xs.max() <= spec["box"]
        assert np.all(small.xs == np.rint(small.xs))
    # clustered configs are far from uniform: occupancy of a 20x20 grid is highly skewed
    c3 = make_config_instance("C3", n=20000)
    h, _, _ = np.histogram2d(c3.xs, c3.ys, bins=20)
    assert h.std() > 1.0 * h.mean()  # uniform C1 gives ~0.15


def test_mode_names():
    assert mode_name(Mode.partial_aco) == "partial" and mode_from_name("classic") == Mode.classic_aco
    assert mode_from_name("nope") is None


# ------------------------------------------------------------------ C ABI

def header_functions():
    text = open(os.path.join(ROOT, "include", "paco_b200.h")).read()
    return sorted(set(re.findall(r"(?:paco_status|void|int|const char\s*\*)\s+(paco_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(native):
    names = header_functions()
    assert set(names) == set(N.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(native):
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_mirror_runconfig(native):
    c = N.Config()
    assert native.paco_config_default(c) == 0
    ref = RunConfig()
    for f in ("ants", "iterations", "alpha", "beta", "partial_prob", "max_mod_frac", "two_opt_prob", "workers",
              "seed", "rho", "tau_max", "tau0", "time_budget_s"):
        assert getattr(c, f) == getattr(ref, f), f


@pytest.mark.parametrize("field,value,msg", [
    ("ants", 0, "ants must be >= 1"), ("iterations", 0, "iterations must be >= 1"),
    ("workers", 0, "workers must be >= 1"), ("partial_prob", 1.5, "partial_prob must be in [0,1]"),
    ("max_mod_frac", 0.0, "max_mod_frac must be in (0,1]"), ("two_opt_prob", -0.1, "two_opt_prob must be in [0,1]"),
    ("rho", 2.0, "rho must be in [0,1]"), ("tau0", 0.0, "tau0 must be positive"),
    ("tau_max", -1.0, "tau_max must be positive"), ("time_budget_s", -1.0, "time budget must be >= 0"),
])
def test_config_validation_messages(native, field, value, msg):
    """RunConfig::validate (engine.hpp:61-75): same checks, same messages, invalid_argument."""
    cfg = RunConfig(**{field: value})
    with pytest.raises(InvalidArgument) as ei:
        cfg.validate()
    assert msg in str(ei.value)


def test_classic_size_limit_and_unsupported(native):
    with pytest.raises(InvalidArgument, match="classic mode requires n <= 5000"):
        RunConfig().validate(n=5001, mode=Mode.classic_aco)
    RunConfig().validate(n=5000, mode=Mode.classic_aco)
    RunConfig(two_opt_prob=0.1, two_opt_window=500).validate()  # f2: supported
    RunConfig(synchronous=False).validate()  # f3: the reference's default async engine
    RunConfig(synchronous=False).validate(mode=Mode.classic_aco)  # classic runs barriered anyway
    with pytest.raises(PacoError) as ei:
        RunConfig(synchronous=False, rule="independent").validate()
    assert ei.value.status == N.PACO_E_UNSUPPORTED
    with pytest.raises(PacoError) as ei:
        RunConfig(synchronous=False, ants=70000).validate()
    assert ei.value.status == N.PACO_E_UNSUPPORTED


def test_no_gpu_fails_loudly(native):
    """The product path has no CPU fallback: without a visible sm_100 GPU, create fails."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    inst = make_config_instance("C1", n=100)
    from paper_1709_03187_b200 import Colony
    with pytest.raises(PacoError) as ei:
        Colony(inst, RunConfig(ants=2))
    assert ei.value.status == N.PACO_E_CUDA


def test_product_does_not_import_oracle():
    """Only tests/, smoke() and bench.py may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_1709_03187_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp")):
                text = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in text and "o2_" not in text and "libo2" not in text, f
    header = open(os.path.join(ROOT, "include", "paco_b200.h")).read()
    assert "o2.h" not in header and "libo2" not in header


def build_drop_in(tmp_dir):
    exe = os.path.join(tmp_dir, "drop_in")
    lib = os.path.dirname(N.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "drop_in.cpp"), "-L", lib, "-lpaco_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


REF_INCLUDE = "/root/reference/proj/include"
REF_DROP_IN = os.path.join(ROOT, "tests", "cpp", "_build", "ref_drop_in")


def build_ref_drop_in(out_path=REF_DROP_IN):
    """tests/cpp/ref_drop_in.cpp against the unmodified reference headers (needs /root/reference;
    __graft_entry__.build() runs this in the build container, the binary travels with the repo)."""
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    lib = os.path.dirname(N.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "ref_drop_in.cpp"), "-L", lib, "-lpaco_b200",
                    f"-Wl,-rpath,{lib}", "-o", out_path], check=True)
    return out_path


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers not present (GPU box)")
def test_cpp_drop_in_on_reference_types_compiles_and_fails_loudly_without_gpu(native, tmp_path):
    """paco_b200::run(const paco::Instance&, const paco::RunConfig&, paco::Mode) -> paco::RunReport
    compiles in one translation unit with the unmodified reference headers;
    the reference's validation errors come through unchanged and, without a GPU, the run
    throws instead of falling back to the CPU."""
    import torch
    exe = build_ref_drop_in(str(tmp_path / "ref_drop_in"))
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu_parity.py::test_cpp_reference_types_drop_in_on_gpu")
    out = subprocess.run([exe, "0"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "no GPU" in out.stdout


def test_cpp_drop_in_header_compiles_and_fails_loudly_without_gpu(native, tmp_path):
    """include/paco_b200/paco.hpp is the reference's C++ calling convention over the C ABI."""
    import torch
    exe = build_drop_in(str(tmp_path))
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu_parity.py::test_cpp_drop_in_on_gpu")
    out = subprocess.run([exe, "0"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "no GPU" in out.stdout


def test_rng_jump_matches_stepping(native):
    """paco_rng_jump (the reference-rule generator's jump: x^J mod the characteristic polynomial
    of the xoshiro256 transition, Cayley-Hamilton) equals J single steps of rng.hpp:40-50."""
    import ctypes

    M = (1 << 64) - 1

    def step(s):
        s = list(s)
        t = (s[1] << 17) & M
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t
        s[3] = ((s[3] << 45) | (s[3] >> 19)) & M
        return s

    for state, steps in (([1, 2, 3, 4], 0), ([1, 2, 3, 4], 1), ([0x9E3779B97F4A7C15, 7, 0, 12345], 64),
                         ([5, 6, 7, 8], 31 * 64), ([11, 22, 33, 44], 12345)):
        inp = (ctypes.c_uint64 * 4)(*state)
        out = (ctypes.c_uint64 * 4)()
        assert native.paco_rng_jump(inp, steps, out) == 0
        ref = state
        for _ in range(steps):
            ref = step(ref)
        assert list(out) == ref, (state, steps)
