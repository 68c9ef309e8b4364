"""The C ABI used from plain C (examples/pnn_example.c): it compiles and links against
libpnn.so here (no GPU needed), and on a B200 it trains, merges and evaluates a PNN."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2304_09590_b200")


def _build(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    exe = str(tmp_path / "pnn_example")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "pnn_example.c"), "-L", LIBDIR, "-lpnn", "-L", "/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.check_call(cmd)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "merged accuracy" in out.stdout
