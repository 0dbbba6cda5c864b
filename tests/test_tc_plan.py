"""Host logic of the tensor-core schedule (paper_2108_12050_b200/csrc/tc_plan.h), on CPU:
window geometry and the block-Toeplitz pair tables read through the kernel's descriptor
addressing (tools/umma_probe.cu confirms the hardware reads them the same way)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tc_plan_tables(tmp_path):
    exe = str(tmp_path / "tc_plan_check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", exe, os.path.join(ROOT, "tests", "cpp", "tc_plan_check.cpp")])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout
