"""The seeded input generators: NumPy and torch agree bit for bit; values are exact bf16."""
import numpy as np
import pytest
import torch

import spa_inputs as si
from oracle.replay import Replay
from spa_inputs import families, workloads


def test_numpy_torch_bit_identical():
    a = si.kv_bits_np(7, si.KIND_K, 12345, [0, 3, 63], np.arange(100, 164), 8, 128)
    b = si.kv_bits_torch(7, si.KIND_K, 12345, [0, 3, 63], np.arange(100, 164), 8, 128, device="cpu")
    assert np.array_equal(a, b.view(torch.int16).numpy().view(np.uint16))


def test_values_exact_and_unit_scale():
    a = si.kv_bits_np(1, si.KIND_V, 3, [0], np.arange(4096), 2, 64)
    f = si.bits_to_f64(a)
    assert np.all(f * 32 == np.round(f * 32)) and np.abs(f).max() <= 3.9375
    assert abs(f.mean()) < 0.01 and 1.1 < f.std() < 1.2


def test_streams_differ():
    a = si.kv_bits_np(1, si.KIND_K, 1, [0], np.arange(64), 2, 64)
    b = si.kv_bits_np(1, si.KIND_K, 2, [0], np.arange(64), 2, 64)
    c = si.kv_bits_np(1, si.KIND_V, 1, [0], np.arange(64), 2, 64)
    assert (a != b).mean() > 0.9 and (a != c).mean() > 0.9


@pytest.mark.parametrize("fam", ["needle_shared_pos", "needle_tail_pos", "needle_cow_pos"])
def test_needles_dominate(fam):
    """The needle families do what they claim: O of the rows they target ~ v[j*]."""
    rec = workloads.random_small(5, workloads.Model("t", 1, 8, 2, 64), max_prefix=120)
    inp = families.make_inputs(rec, fam)
    rp = Replay(inp)
    O, _ = rp.expected(0, inp.q[0])
    assert inp.needles
    G = 4
    for key, pos in inp.needles.items():
        if key[0] == "group":
            gi = key[1]
            names = [nm for nm in inp.batch if nm[0] == gi]
            origin = (gi, "main")
        else:
            names = [key[1]]
            origin = key[1]
        for nm in names:
            i = inp.batch.index(nm)
            v = families._poscode_v(families.origin_id(origin), [pos], 2, 64)
            vf = si.bits_to_f64(v)[0]
            for h in range(8):
                assert np.abs(O[i, h] - vf[h // G]).max() < 2e-3
