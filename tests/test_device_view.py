"""DeviceView (the reference's in-place state arrays over device tensors) on CPU
tensors: reads copy, item assignment writes through, numpy interop works the way
the reference's callers use the arrays (field.py:47-58, batch.py:240-243,
tests/test_acceptance.py:234-249 of the reference)."""

import numpy as np
import torch

from paper_2505_00690_b200.crowd import DeviceView


def test_reads_and_numpy_interop():
    t = torch.arange(12, dtype=torch.float64).reshape(2, 3, 2)
    v = DeviceView(t)
    a = np.asarray(v)
    assert a.shape == (2, 3, 2) and v.shape == (2, 3, 2) and v.dtype == np.float64
    assert np.array_equal(v, t.numpy())
    assert np.array_equal(v + 1, t.numpy() + 1) and np.array_equal(1 - v, 1 - t.numpy())
    assert float(v[1, 2, 0]) == 10.0
    assert np.array_equal(np.hypot(*v[0, 1]), np.hypot(2.0, 3.0))
    assert np.array_equal(v.copy(), t.numpy()) and v.sum() == t.sum().item()
    assert np.array_equal(np.stack([v, v]), np.stack([t.numpy(), t.numpy()]))
    assert np.array_equal((v[:, :, None, :] - v[:, None, :, :]).shape, (2, 3, 3, 2))


def test_item_assignment_writes_through():
    t = torch.zeros((2, 3, 2), dtype=torch.float64)
    v = DeviceView(t)
    v[0, 1] = [3.5, 4.5]
    assert t[0, 1].tolist() == [3.5, 4.5]
    v[1][2] = (1.0, 2.0)                 # chained basic indexing is a view of the tensor
    assert t[1, 2].tolist() == [1.0, 2.0]
    v[:, :, 0] += 0.5                    # augmented assignment through __setitem__
    assert t[0, 0, 0].item() == 0.5
    v[np.array([0, 1]), 0] = np.array([[9.0, 9.0], [8.0, 8.0]])
    assert t[0, 0].tolist() == [9.0, 9.0] and t[1, 0].tolist() == [8.0, 8.0]
    w = v[np.array([0])]                 # advanced indexing copies, as in numpy
    w[0, 0] = [-1.0, -1.0]
    assert t[0, 0].tolist() == [9.0, 9.0]


def test_bool_view():
    t = torch.tensor([[1, 0, 1]], dtype=torch.uint8)
    v = DeviceView(t, bool)
    assert np.asarray(v).dtype == bool and v.sum() == 2
    v[0, 1] = True
    assert t.tolist() == [[1, 1, 1]]
    assert bool(v[0, 2]) is True
