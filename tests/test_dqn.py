"""Device double-DQN update: rs_dqn_update(_host)
against the compiled reference's own DqnAgent::update (oracle/_ref,
ref_dqn_train) — loss and every online parameter bitwise after every step,
target-network sync included.  The batch each step draws is read back from
the reference (ReplayBuffer::sample with the same Rng), so both sides
differentiate the same samples in the same order."""
import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine


def transitions(dim, actions, n, seed):
    rng = np.random.default_rng(seed)
    s = rng.random((n, dim))
    s[s < 0.3] = 0.0                      # encode_state has many exact zeros
    ns = rng.random((n, dim))
    ns[ns < 0.3] = 0.0
    a = rng.integers(0, actions, n)
    r = rng.normal(size=n) * 3.0          # includes |e| > 1 (Huber's linear branch)
    d = rng.random(n) < 0.05
    return s, a, r, ns, d


def test_dqn_abi_structs():
    import ctypes as C
    assert C.sizeof(abi.DqnBatch) == 8 + 5 * 8
    assert C.sizeof(abi.DqnState) == 4 * 8 + 3 * 8 + 8


@pytest.mark.skipif(not O.have_ref(), reason="compiled reference unavailable")
def test_reference_dqn_driver_runs():
    dims = [27, 64, 64, 5]
    p = O.ref_agent_params(27, 5, 64, 42)
    s, a, r, ns, d = transitions(27, 5, 300, 1)
    idx, loss, online, target = O.ref_dqn_train(dims, p, s, a, r, ns, d, 64, 3, 5, 0.9)
    assert idx.shape == (3, 64) and len(set(idx[0])) == 64   # without replacement
    assert np.all(loss > 0) and not np.array_equal(online[-1], p)


@pytest.mark.gpu
@pytest.mark.skipif(not O.have_ref(), reason="compiled reference unavailable")
@pytest.mark.parametrize("m,hidden,batch,steps,sync", [(4, 64, 512, 4, 2), (8, 64, 128, 3, 1000),
                                                       (2, 32, 7, 5, 3)])
def test_gpu_dqn_update_matches_reference(m, hidden, batch, steps, sync):
    dim = abi.state_dimension(m)
    dims = [dim, hidden, hidden, m + 1]
    p = O.ref_agent_params(dim, m + 1, hidden, 42)
    s, a, r, ns, d = transitions(dim, m + 1, batch + 90, m)
    discount = 0.5 * 0.99
    idx, loss, online, target = O.ref_dqn_train(dims, p, s, a, r, ns, d, batch, steps, 11,
                                                discount, sync_interval=sync)
    tr = engine.DqnTrainer(dims, p, target_sync_interval=sync)
    for k in range(steps):
        j = idx[k]
        got = tr.update(s[j], a[j], r[j], ns[j], d[j], discount)
        assert np.float64(got).view(np.uint64) == loss[k].view(np.uint64), (k, got, loss[k])
        bad = tr.online.view(np.uint64) != online[k].view(np.uint64)
        assert not bad.any(), (k, int(bad.sum()), int(np.flatnonzero(bad)[0]))
    assert np.array_equal(tr.target.view(np.uint64), target.view(np.uint64))
    assert tr.updates == steps and tr.adam_t == steps
