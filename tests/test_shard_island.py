"""CPU: the closed-form island-match count of shard_moves (common.cuh
island_matches) equals the reference's unit-by-unit pairing
(placement.hpp:88-97) on random device sets over contiguous islands."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_island_matches_equal_unit_pairing(tmp_path):
    exe = tmp_path / "shard_island"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-I", str(ROOT / "include"), "-o", str(exe),
                    str(ROOT / "tests" / "native" / "shard_island.cu")], check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert " 0 mismatches" in out.stdout
