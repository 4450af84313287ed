"""The C-ABI libraries load and export every symbol their headers declare;
no compute without a GPU (the product path has no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hb(?:gpu|o)_[a-z0-9_]+)\s*\(", text)))


def exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True)
    return {line.split()[-1] for line in out.stdout.splitlines() if line.strip()}


def test_libhbgpu_exports_header():
    so = os.path.join(ROOT, "paper_2411_14315_b200", "libhbgpu.so")
    names = declared(os.path.join(ROOT, "include", "hbgpu.h"))
    assert len(names) >= 30
    syms = exported(so)
    missing = [n for n in names if n not in syms]
    assert not missing, missing
    lib = ctypes.CDLL(so)
    for n in names:
        getattr(lib, n)


def test_oracle_restatement_exports_header():
    so = os.path.join(ROOT, "oracle", "_ref", "libhboracle.so")
    names = declared(os.path.join(ROOT, "oracle", "hbgls_oracle.h"))
    syms = exported(so)
    assert not [n for n in names if n not in syms]


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_14315_b200 import hbgpu, meshgen

    mesh = meshgen.hex_cylinder(0.3, 1.0, 2, 2, 2)
    with pytest.raises(hbgpu.CudaError, match="no CPU fallback"):
        hbgpu.GpuContext(mesh)


def test_product_does_not_import_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_2411_14315_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".hpp")) or f == "Makefile":
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                bad = re.findall(r"import oracle|from oracle|oracle/_ref|oracle\.bindings|libhbref|libhboracle",
                                 text)
                assert not bad, (f, bad)
