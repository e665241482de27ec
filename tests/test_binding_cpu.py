"""Host-side checks of the Python binding and FastronModel that need no GPU: argument
validation before any library call (dtype, inner contiguity, float4 records), and the
checkpoint's robot-identity check."""
import numpy as np
import pytest
import torch

import workloads as W


def test_expect_rejects_wrong_dtype_and_strides():
    import paper_1910_06451_b200 as fb
    q = torch.zeros((10, 7), dtype=torch.float64)
    with pytest.raises(ValueError, match="float32"):
        fb._expect(q, torch.float32, "q", dim=2)
    qt = torch.zeros((7, 10), dtype=torch.float32).t()  # transposed: stride(1) != 1
    with pytest.raises(ValueError, match="contiguous"):
        fb._expect(qt, torch.float32, "q", dim=2)
    fb._expect(torch.zeros((10, 7), dtype=torch.float32)[:, :5], torch.float32, "q", dim=2)  # ld > D is fine
    with pytest.raises(ValueError, match="dimensions"):
        fb._expect(torch.zeros(5, dtype=torch.float32), torch.float32, "q", dim=2)


def test_expect_pos_layout():
    import paper_1910_06451_b200 as fb
    fb._expect_pos(torch.zeros((8, 100, 4), dtype=torch.float32), "pos", 8)
    fb._expect_pos(torch.zeros((8, 120, 4), dtype=torch.float32)[:, :100], "pos", 8)  # ldpos > n
    with pytest.raises(ValueError):
        fb._expect_pos(torch.zeros((8, 100, 3), dtype=torch.float32), "pos")
    with pytest.raises(ValueError):
        fb._expect_pos(torch.zeros((100, 8, 4), dtype=torch.float32).transpose(0, 1), "pos")
    with pytest.raises(ValueError):
        fb._expect_pos(torch.zeros((8, 100, 4), dtype=torch.float32), "pos", 16)
    with pytest.raises(ValueError):
        fb._expect_pos(torch.zeros((8, 100, 4), dtype=torch.float64), "pos")


def _state(robot, **over):
    st = {"supports": torch.zeros((3, robot.dof)), "alpha": torch.zeros(3, dtype=torch.float64),
          "labels": torch.ones(3, dtype=torch.int8), "kind": 0, "gamma": 5.0, "beta": 1.0,
          "robot_dh": torch.as_tensor(np.asarray(robot.dh, dtype=np.float32)),
          "robot_cp_frame": torch.as_tensor(np.asarray(robot.cp_frame, dtype=np.int32)),
          "robot_cp_offset": torch.as_tensor(np.asarray(robot.cp_offset, dtype=np.float32)),
          "robot_base": torch.as_tensor(np.asarray(robot.base, dtype=np.float32))}
    st.update(over)
    return st


@pytest.mark.parametrize("field", ["robot_dh", "robot_cp_frame", "robot_cp_offset", "robot_base"])
def test_checkpoint_of_another_robot_is_rejected(field):
    """Every robot quantity the scores depend on must match before a checkpoint loads."""
    from paper_1910_06451_b200.model import FastronModel
    r = W.arm7(8)
    st = _state(r)
    v = st[field].clone()
    if field == "robot_cp_frame":
        v[0] = (int(v[0]) + 1) % (r.dof + 1)
    else:
        v.view(-1)[0] += 0.01
    st[field] = v
    with pytest.raises(ValueError, match=field):
        FastronModel(r).load_state_dict(st, device="cpu")
