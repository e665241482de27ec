"""Optional content validation of the C ABI (include/fastron.h conventions):
with validation on, non-finite inputs and labels outside {-1, +1} are rejected with
FASTRON_ERR_INVALID_ARG before any computation; valid inputs run unchanged."""
import numpy as np
import pytest

import workloads as W
from gpu_helpers import dev, require_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture
def validating():
    import paper_1910_06451_b200 as fb
    before = fb.validation()
    fb.set_validation(True)
    yield fb
    fb.set_validation(before)


def test_nonfinite_configuration_rejected(validating):
    require_gpu()
    fb = validating
    robot = W.arm7(8)
    q = W.uniform_configs(np.random.default_rng(0), 100, 7)
    pos = fb.fastron_fk(robot, dev(q))  # valid: runs
    q[37, 3] = np.nan
    with pytest.raises(fb.FastronError) as e:
        fb.fastron_fk(robot, dev(q))
    assert e.value.status == fb.FASTRON_ERR_INVALID_ARG and "non-finite" in str(e.value)
    alpha = np.ones(100, np.float32)
    alpha[5] = np.inf
    with pytest.raises(fb.FastronError):
        fb.fastron_score(pos, pos, dev(alpha), 0, 5.0)


def test_bad_labels_rejected(validating):
    require_gpu()
    import torch
    fb = validating
    robot = W.arm7(8)
    q = W.uniform_configs(np.random.default_rng(1), 64, 7)
    pos = fb.fastron_fk(robot, dev(q))
    K = fb.fastron_gram(pos, 0, 5.0)
    y = torch.ones(64, dtype=torch.int8, device="cuda")
    y[::2] = -1
    fb.fastron_train(K, y, 1.0, 100, 64)  # valid: runs
    y[10] = 0
    with pytest.raises(fb.FastronError) as e:
        fb.fastron_train(K, y, 1.0, 100, 64)
    assert e.value.status == fb.FASTRON_ERR_INVALID_ARG and "labels" in str(e.value)
