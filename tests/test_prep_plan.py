"""Host-side plans of the union metadata kernel (no GPU needed): tools/prep_plan_check.cu compiles prep.cuh with nvcc
and checks on the CPU that every (block, part) of the prep kernel's CTA plans — densest-blocks-first and the
overlapped (window-major, split tail) variant — is produced exactly once with consecutive ids, and the UP raster-group
rule's range."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
def test_prep_plans(tmp_path):
    exe = tmp_path / "prep_plan_check"
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "--expt-relaxed-constexpr", "-o",
                    str(exe), os.path.join(ROOT, "tools", "prep_plan_check.cu")], check=True, capture_output=True,
                   timeout=300)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-3000:]
