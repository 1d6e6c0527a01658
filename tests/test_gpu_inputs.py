"""Device-side seeded inputs are bitwise equal to the numpy spec."""

import numpy as np
import pytest

from paper_1710_01839_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tok,wide,shape,seed", [("dd", False, (37, 45, 29), 0),
                                                 ("dd", True, (64, 33, 70), 12),
                                                 ("qd", False, (21, 19, 23), 13),
                                                 ("dd", False, (1024, 1024, 1024), 0),
                                                 ("qd", False, (512, 300, 260), 1)])
def test_device_inputs_bitwise_equal_host(gpu, tok, wide, shape, seed):
    a, b = inputs.gemm_inputs(tok, *shape, seed=seed, wide=wide)
    da, db = inputs.gemm_inputs_device(tok, *shape, seed=seed, wide=wide)
    assert np.array_equal(da.cpu().numpy(), a)
    assert np.array_equal(db.cpu().numpy(), b)
    assert (da.cpu().numpy().view(np.uint64) == a.view(np.uint64)).all()   # bit patterns too
