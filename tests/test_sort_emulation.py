"""CPU: the device-side libstdc++ std::sort emulation (common.cuh ls_sort),
compiled for the host, reproduces std::sort's permutation and comparator call
sequence on tie-heavy inputs."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_ls_sort_matches_libstdcxx(tmp_path):
    exe = tmp_path / "sort_emul"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-I", str(ROOT / "include"), "-o", str(exe),
                    str(ROOT / "tests" / "native" / "sort_emul.cu")], check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "0 mismatches" in out.stdout
