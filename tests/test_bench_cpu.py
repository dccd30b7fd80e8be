"""bench.py host logic on CPU: the reference arm's JSON line (CPU restatement on
a bounded sample) and the e2e copy-group split."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def test_e2e_groups_partition_layers():
    import bench
    for L in (1, 2, 5, 32, 80):
        for cuts in ([1, 4], [L // 2, L - 4, L - 1]):
            groups = bench.e2e_groups(L, cuts)
            assert [l for g in groups for l in g] == list(range(L))
            assert all(g for g in groups)
    assert bench.e2e_groups(32, [16, 28, 31])[-1] == [31]


def test_role_runs_cover_baseline_and_offload():
    import bench
    assert (0.0, False) in bench.ROLE_RUNS
    assert any(r > 0 and not zc for r, zc in bench.ROLE_RUNS)
    assert any(zc for _, zc in bench.ROLE_RUNS)


@pytest.mark.usefixtures("built")
def test_reference_arm_line(tmp_path):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--config", "C1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, cwd=tmp_path)
    assert r.returncode == 0, r.stderr[-500:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
