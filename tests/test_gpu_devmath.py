"""The fp64 building blocks of the covariance generation (csrc/mra_device.cuh: exp_neg, sqrt_fast, covf)
against libm on the device, on dense grids of 1e8-2e8 arguments (tools/check_exp.cu)."""
import os
import re
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exp_sqrt_covf_accuracy(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "check_exp"
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           os.path.join(ROOT, "tools", "check_exp.cu"), "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True, timeout=300).stdout
    ulps = [float(v) for v in re.findall(r"exp_neg .*max ([0-9.]+) ulp", out)]
    assert len(ulps) == 3 and max(ulps) <= 1.5, out
    sq = float(re.search(r"sqrt_fast vs .*max ([0-9.]+) ulp", out).group(1))
    assert sq <= 1.0, out
    tiny = re.search(r"sqrt_fast tiny .*max ([0-9.]+) ulp; special cases failed: (\d+)", out)
    assert float(tiny.group(1)) <= 1.0 and int(tiny.group(2)) == 0, out
    rel = [float(v) for v in re.findall(r"covf kind \d .*max relative ([0-9.e+-]+)", out)]
    assert len(rel) == 2 and max(rel) <= 1e-14, out
