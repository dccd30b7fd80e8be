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
    assert set(bench.CAPACITY_RUNS) == {"C4", "C5"}


def test_capacity_cases_plan_a_larger_offloaded_batch():
    """The capacity cases behind the N > 1 comparison: under each case's memory
    policy the offloaded steady-state batch is larger than the local-only one
    (C4 planner bound, C5 bound 0.7), at full and at the 1-GPU scaled budgets."""
    from paper_2503_20552_b200 import capacity, config, specs
    for name, case in capacity.CAPACITY_CASES.items():
        for nd in (1, 2, 4):
            cfg = config.SimConfig(gpu=specs.B200, model=case.model, num_prefill=nd,
                                   num_decode=nd, offload_ratio=case.offload_ratio)
            reqs = capacity.case_requests(case, 0)
            for scale in (1.0, 0.45):
                plan = capacity.plan_capacity(cfg, reqs, scale=scale)
                assert plan.batch_offload > plan.batch_no_offload > 0, (name, nd, scale)
                assert plan.bytes("no_offload") <= plan.pool_bytes
                assert plan.bytes("local") <= plan.pool_bytes
                assert plan.bytes("offloaded") <= plan.exec_budget_bytes


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


def _role_runs_worker(rank, world, port, out):
    import os
    from types import SimpleNamespace
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    bench.ROLE_RUNS = ((0.0, False),)  # one role run and one capacity run exercise the plumbing
    bench.CAPACITY_RUNS = ("C5",)
    args = SimpleNamespace(role_config="C1", role_timeout=120.0)
    res = bench.role_split_runs(args, world, rank)
    if rank == 0:
        out.put(res)
    dist.destroy_process_group()


def test_role_split_runs_are_isolated_on_failure():
    """N > 1 orchestration: rank 0 launches the role split as its own torchrun
    while the main ranks wait on a CPU barrier; a run that cannot work (no GPU
    here) comes back as an error entry instead of taking the main line down."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_role_runs_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res) == 2 and res[0]["offload_ratio"] == 0.0 and res[0]["exchange"] == "nccl"
    assert res[1]["capacity"] == "C5"
    assert all("error" in r or "tokens_per_s" in r or "value" in r for r in res)
