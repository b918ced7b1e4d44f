"""C-ABI boundary checks that need no GPU: libunocg.so loads and exports every entry point
declared in include/*.h (uno_cg.h, uno_cg_slab.h); the ctypes structs match the C layout;
argument validation paths that fail before touching the device return the documented
status codes."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDRS = [os.path.join(ROOT, "include", f) for f in sorted(os.listdir(os.path.join(ROOT, "include"))) if f.endswith(".h")]
LIB = os.path.join(ROOT, "paper_2508_02681_b200", "lib", "libunocg.so")


def _ensure_built():
    if not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    assert os.path.exists(LIB)


def _declared():
    txt = "".join(open(h).read() for h in HDRS)
    return sorted(set(re.findall(r"\b(uno_(?:cg|slab)_[A-Za-z_]+)\s*\(", txt)) - {"uno_cg_handle", "uno_slab_handle"})


def test_header_declares_north_star_entry_points():
    names = _declared()
    for n in ("uno_cg_create", "uno_cg_apply_K", "uno_cg_apply_precond", "uno_cg_solve", "uno_cg_effective_property"):
        assert n in names


def test_library_exports_every_declared_symbol():
    _ensure_built()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT\s+(uno_(?:cg|slab)_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert "uno_slab_create" in exported and "uno_slab_kapply" in exported
    # nothing but the C ABI is exported (hidden visibility for the C++/CUDA internals)
    extra = [l for l in out.splitlines()
             if " T " in l and "uno_cg_" not in l and "uno_slab_" not in l and "_init" not in l and "_fini" not in l]
    assert not extra, extra[:5]


def test_library_loads_and_validates_without_gpu():
    _ensure_built()
    import torch  # noqa: F401  (makes libcudart resolvable)

    from paper_2508_02681_b200 import binding as B

    assert B.uno_cg_version().startswith("libunocg")
    # struct layout matches the header (offsets checked against the C declaration order)
    assert ctypes.sizeof(B.UnoCgDesc) == 120
    assert B.UnoCgDesc.stream.offset == 112 and B.UnoCgDesc.seed.offset == 88
    assert ctypes.sizeof(B.UnoCgReport) == 40
    d = B.UnoCgDesc()
    d.dim = 4
    with pytest.raises(B.UnoError) as e:
        B.uno_cg_create(d, 1)
    assert e.value.status == B.UNO_ERR_ARG
    d.dim, d.n[0], d.n[1], d.n[2], d.nrhs = 3, 12, 8, 8, 1
    d.mat[0][0] = d.mat[1][0] = 1.0
    with pytest.raises(B.UnoError) as e:
        B.uno_cg_create(d, 1)
    assert e.value.status == B.UNO_ERR_SHAPE
    d.n[0] = 16
    d.bc[0] = 1  # Dirichlet on x only: not one of the built boundary patterns
    with pytest.raises(B.UnoError) as e:
        B.uno_cg_create(d, 1)
    assert e.value.status == B.UNO_ERR_UNSUPPORTED
    with pytest.raises(B.UnoError) as e:
        B.uno_cg_workspace_size(d)
    assert e.value.status == B.UNO_ERR_UNSUPPORTED
    d.bc[0] = 0
    with pytest.raises(B.UnoError) as e:  # misaligned caller workspace, rejected before any device work
        B.uno_cg_create(d, 1, 8)
    assert e.value.status == B.UNO_ERR_ARG


def test_workspace_size_accounts_for_the_cg_state():
    _ensure_built()
    import torch  # noqa: F401

    from paper_2508_02681_b200 import binding as B

    d = B.UnoCgDesc()
    d.dim, d.n[0], d.n[1], d.n[2], d.nrhs = 3, 256, 256, 256, 3
    d.mat[0][0], d.mat[1][0] = 1.0, 100.0
    n = 256 ** 3
    ws = B.uno_cg_workspace_size(d)
    vec = 3 * n * 8
    spec = 3 * 129 * 256 * 256 * 16
    gtab = 129 * 256 * 256 * 8
    # r, d, d2 (second direction buffer of the paired u updates), p, u + spectrum + G_hat + small
    assert 5 * vec + spec + gtab <= ws <= 5 * vec + spec + gtab + (64 << 20)
    assert ws % 256 == 0
    d.physics, d.nrhs = 1, 1  # elastic: 3 components, 6 symbol planes
    d.mat[0][1] = d.mat[1][1] = 1.0
    ws_e = B.uno_cg_workspace_size(d)
    assert ws_e >= 4 * 3 * n * 8 + 3 * 129 * 256 * 256 * 16 + 6 * 129 * 256 * 256 * 8


def test_slab_create_validates_without_gpu():
    _ensure_built()
    import torch  # noqa: F401

    from paper_2508_02681_b200 import binding as B

    d = B.UnoCgDesc()
    d.dim, d.n[0], d.n[1], d.n[2], d.nrhs = 2, 32, 32, 1, 1
    d.mat[0][0] = d.mat[1][0] = 1.0
    with pytest.raises(B.UnoError) as e:
        B.uno_slab_create(d, 0, 2, 1)
    assert e.value.status == B.UNO_ERR_UNSUPPORTED  # slab mode: 3D only
    d.dim, d.n[2] = 3, 24
    with pytest.raises(B.UnoError) as e:
        B.uno_slab_create(d, 0, 2, 1)
    assert e.value.status == B.UNO_ERR_SHAPE  # N3 not a power of two
    d.n[2] = 32
    with pytest.raises(B.UnoError) as e:
        B.uno_slab_create(d, 2, 2, 1)
    assert e.value.status == B.UNO_ERR_ARG  # rank out of range
