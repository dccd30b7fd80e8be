"""The command line on CPU: `run` with analytic pricing reproduces simulate()."""
import json

from paper_2503_20552_b200 import cli, config, engine, workload


def test_cli_run_matches_simulate(tmp_path, capsys):
    cfg = {"num_prefill": 2, "num_decode": 2, "offload_ratio": 0.5}
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    assert cli.main(["run", "--config", str(p), "--rate", "6", "--requests", "80", "--seed", "3"]) == 0
    out = json.loads(capsys.readouterr().out)
    r = engine.simulate(config.SimConfig.from_dict(cfg),
                        workload.synth_requests(workload.preset("sharegpt_like", 6.0, 80), 3))
    assert out["pricer"] == "analytic" and out["completed"] == 80
    assert out["end_time_s"] == r.end_time and out["steps"] == len(r.steps)
    assert out["bound"] == 0.5


def test_cli_run_trace_and_offload_override(tmp_path, capsys):
    reqs = workload.synth_requests(workload.preset("long_prompt", 2.0, 20), 1)
    trace = tmp_path / "t.jsonl"
    workload.save_trace_jsonl(trace, reqs)
    assert cli.main(["run", "--trace", str(trace), "--offload-ratio", "0"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["completed"] == 20 and out["offloaded_slot_share"] == 0.0


def test_bmax_fit_and_gpu_override():
    """B_max by sweep: the knee of t(B) = max(t0, t0 B / B_max) is recovered from
    noisy samples, and the GpuSpec override makes the reference formula
    (costs.b_max) return it."""
    import random

    from paper_2503_20552_b200 import bmax, costs, specs
    rng = random.Random(0)
    knee, t0 = 173.0, 1e-4
    samples = [(b, max(t0, t0 * b / knee) * (1 + 0.01 * rng.uniform(-1, 1)))
               for b in (1, 8, 16, 32, 64, 128, 192, 256, 384, 512, 1024)]
    ft0, fk = bmax.fit_knee(samples)
    assert abs(ft0 - t0) / t0 < 0.02 and abs(fk - knee) / knee < 0.03
    for k in (1, 17, 132, 173, 900):
        gpu = bmax.gpu_for_bmax(specs.B200, specs.LLAMA2_7B, k)
        assert costs.b_max(gpu, specs.LLAMA2_7B) == k
    # flat everywhere: the largest batch is a lower bound
    assert bmax.fit_knee([(1, 1.0), (64, 1.0), (256, 1.05)])[1] == 256.0
