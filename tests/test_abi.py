"""C-ABI library checks that need no GPU: it loads, exports every symbol
declared in include/*.h, the host setup works, and compute entry points
refuse to run without a device (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from paper_2205_04401_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("vp.h", "vp_setup.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*(vps?_[a-z0-9_]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 20
    L = ctypes.CDLL(_lib.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), f"{n} declared in include/ but not exported"
    assert names == set(_lib.SYMBOLS), "python binding out of sync with the headers"


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="a GPU is present")
def test_no_cpu_fallback_without_device():
    with pytest.raises(vp.DeviceError):
        vp.Evaluator(0)
    h = ctypes.c_void_p()
    assert _lib.lib().vp_create(0, ctypes.byref(h)) == 3


@pytest.mark.parametrize("cfg,n_tri,n_tgt,p,q", [(1, 512, 7680, 4, 6), (2, 4096, 184320, 8, 16),
                                                 (4, 1048576, 29360128, 6, 12)])
def test_config_sizes(cfg, n_tri, n_tgt, p, q):
    I = vp.config_info(cfg)
    assert (I["n_tri"], I["n_tgt"], I["p"], I["q"]) == (n_tri, n_tgt, p, q)


def test_star_configs_near_nominal_size():
    assert abs(vp.config_info(3)["n_tri"] - 65536) / 65536 < 0.02
    assert abs(vp.config_info(5)["n_tri"] - 262144) / 262144 < 0.02
    assert vp.config_info(5, q_override=24)["q"] == 24


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_config_meshes_are_valid(cfg):
    pr = vp.load_config(cfg, with_rules=False)
    P = pr.vxy[pr.tri]
    det = (P[:, 1, 0] - P[:, 0, 0]) * (P[:, 2, 1] - P[:, 0, 1]) - (P[:, 2, 0] - P[:, 0, 0]) * (P[:, 1, 1] - P[:, 0, 1])
    assert (det > 0).all()
    # total area: square 1, polygonal disk < pi, star ~ int r_b^2/2
    area = det.sum() / 2
    if cfg == 1:
        assert abs(area - 1.0) < 1e-12
    elif cfg == 2:
        assert 3.1 < area < np.pi
    # every edge shared by at most two triangles
    e = np.sort(np.concatenate([pr.tri[:, [0, 1]], pr.tri[:, [1, 2]], pr.tri[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    assert cnt.max() <= 2
    assert np.isfinite(pr.coeffs).all()


def test_configs_are_seed_deterministic():
    a = vp.load_config(1, seed=0, with_rules=False)
    b = vp.load_config(1, seed=0, with_rules=False)
    c = vp.load_config(1, seed=1, with_rules=False)
    assert np.array_equal(a.vxy, b.vxy) and np.array_equal(a.coeffs, b.coeffs)
    assert not np.array_equal(a.vxy, c.vxy)


def test_density_projection_reproduces_polynomials():
    vxy = np.array([[0.0, 0.0], [1.0, 0.2], [0.1, 0.9]])
    tri = np.array([[0, 1, 2]], dtype=np.int32)
    co = vp.project_density(vxy, tri, 1, vp.F_LINEAR, [0.5, 2.0, -1.0])
    from oracle import binding as ob
    for xi, eta in [(0.2, 0.3), (0.0, 0.0), (0.6, 0.1)]:
        y = vxy[0] + xi * (vxy[1] - vxy[0]) + eta * (vxy[2] - vxy[0])
        f = co[0] @ ob.koornwinder(1, xi, eta)
        assert abs(f - (0.5 + 2.0 * y[0] - 1.0 * y[1])) < 1e-14


def header_struct_fields(header, typedef_name):
    """Field names, in order, of `typedef struct { ... } typedef_name;` in include/."""
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    m = re.search(r"typedef struct\s*\{([^}]*)\}\s*" + typedef_name + r"\s*;", src)
    assert m, f"{typedef_name} not found in {header}"
    names = []
    for decl in m.group(1).split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.split(","):  # "double a, b" style declarations
            names.append(re.sub(r"\[.*\]", "", part).strip().split()[-1].lstrip("*"))
    return names


@pytest.mark.parametrize("header,name,cls", [("vp.h", "vp_stats", "VpStats"), ("vp.h", "vp_rules", "VpRules")])
def test_ctypes_structs_mirror_headers(header, name, cls):
    """The ctypes mirrors of the C-ABI structs list the header's fields in the
    header's order (a field added on one side only shifts every later one)."""
    fields = [f for f, _ in getattr(_lib, cls)._fields_]
    assert fields == header_struct_fields(header, name)


def test_cpp_caller_builds_and_refuses_without_device():
    """A plain C++ program links libvp_b200.so through include/*.h only
    (tests/cpp/vp_abi_caller.cpp, the reference-side binding of INTEGRATION.md);
    without a GPU it stops with status 3 (no CPU fallback)."""
    import subprocess
    r = subprocess.run(["make", "-C", ROOT, "abi-caller"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    exe = os.path.join(ROOT, "tests", "cpp", "vp_abi_caller")
    assert os.path.exists(exe)
    if _has_gpu():
        pytest.skip("a GPU is present (run by tests/test_gpu_r02.py)")
    r = subprocess.run([exe, "/tmp/vp_abi_caller_u.bin"], capture_output=True, text=True)
    assert r.returncode == 3, (r.returncode, r.stderr)


def test_fmm_order_for_tolerance():
    """eps_fmm -> order: monotone, p + 1 a multiple of four in
    [8, 32], the default order at the evaluation tolerance."""
    orders = [vp.fmm_order_for(e) for e in (1e-1, 1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12, 1e-14, 1e-30)]
    assert orders == sorted(orders)
    assert all((p + 1) % 4 == 0 and 7 <= p <= 31 for p in orders)
    assert orders[0] == 7 and vp.fmm_order_for(1e-8) == 19 and vp.fmm_order_for(1e-12) == 31 and orders[-1] == 31
    assert vp.fmm_order_for(0.0) == 31 and vp.fmm_order_for(float("nan")) == 31
