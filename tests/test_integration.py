"""The header-only qdwh:: adapter (include/qdwhg_qdwh_adapter.hpp) compiles
against the untouched reference headers and links against libqdwhg.so (CPU);
the prebuilt demo gives the reference's answers through libqdwhg (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/core/include"
DEMO = os.path.join(ROOT, "oracle", "_ref", "adapter_demo")


def build_demo():
    lib = os.path.join(ROOT, "paper_2104_14186_b200", "lib")
    ref = os.path.join(ROOT, "oracle", "_ref")
    cmd = ["g++", "-std=c++20", "-O2", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "adapter_demo.cpp"), "-o", DEMO,
           "-L", lib, "-lqdwhg", "-L", ref, "-lqdwhref",
           f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{ref}",
           "-Wl,-rpath,$ORIGIN/../../paper_2104_14186_b200/lib", "-Wl,-rpath,$ORIGIN"]
    subprocess.check_call(cmd)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not mounted")
def test_adapter_compiles_against_reference_headers():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libqdwhref.so")):
        pytest.skip("oracle/_ref not built")
    build_demo()
    assert os.path.exists(DEMO)


@pytest.mark.gpu
def test_adapter_demo_runs(cuda):
    if not os.path.exists(DEMO):
        pytest.skip("adapter demo not prebuilt (needs the reference headers at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr
