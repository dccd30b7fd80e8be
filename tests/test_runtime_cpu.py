"""Host logic of the measured pricer on CPU: a step timed as on two GPUs (the
decoder's local attention alone, the executor's side alone beside the prefill
load) stalls per layer by max(0, remote path - local attention), the
reference's composition (engine.py:441-456)."""
import pytest

from paper_2503_20552_b200.runtime import StepTimes, two_sided_step


def test_two_sided_step_stalls_per_layer():
    loc = StepTimes(total=3e-3, local_attn=3e-3, per_layer_local=[1e-3, 2e-3])
    rem = StepTimes(total=4e-3, exec_attn=2.5e-3, link_bytes=4096,
                    per_layer_stall=[1.5e-3, 1.0e-3])  # the remote path of each layer
    t = two_sided_step(loc, rem)
    assert t.per_layer_stall == pytest.approx([0.5e-3, 0.0])
    assert t.stall == pytest.approx(0.5e-3)
    assert t.local_attn == loc.local_attn and t.exec_attn == rem.exec_attn
    assert t.link_bytes == 4096
    assert t.total == pytest.approx(3.5e-3)


def test_two_sided_step_needs_matching_layers():
    with pytest.raises(ValueError):
        two_sided_step(StepTimes(per_layer_local=[1e-3]), StepTimes(per_layer_stall=[1e-3, 1e-3]))
