"""``LMS.tune_windows`` under DDP trains nothing: its trial steps run the local
replica and the weights, buffers and optimizer state are put back afterwards
(``torch_lms._snapshot_training_state`` / ``_restore_training_state``), so DP
replicas stay identical however many trial steps each took."""

import torch

from paper_1807_02037_b200.torch_lms import _restore_training_state, _snapshot_training_state


def _train(m, o, x, n):
    for _ in range(n):
        o.zero_grad()
        m(x).sum().backward()
        o.step()


def _state(m, o):
    return ([t.clone() for t in (*m.parameters(), *m.buffers())],
            {i: {k: (v.clone(), v.device) if torch.is_tensor(v) else v for k, v in st.items()}
             for i, (_, st) in enumerate(o.state.items())})


def test_restore_round_trip_sgd_and_adam():
    torch.manual_seed(0)
    x = torch.randn(8, 4)
    for make in (lambda p: torch.optim.SGD(p, lr=0.1, momentum=0.9), lambda p: torch.optim.Adam(p, lr=0.1)):
        m = torch.nn.Sequential(torch.nn.Linear(4, 4), torch.nn.BatchNorm1d(4))
        o = make(m.parameters())
        _train(m, o, x, 1)
        before = _state(m, o)
        snap = _snapshot_training_state(m, o)
        _train(m, o, x, 3)
        _restore_training_state(m, o, snap)
        after = _state(m, o)
        assert all(torch.equal(a, b) for a, b in zip(before[0], after[0]))
        for i, st in before[1].items():
            for k, v in st.items():
                w = after[1][i][k]
                if isinstance(v, tuple):
                    assert torch.equal(v[0], w[0]) and v[1] == w[1], k   # Adam's CPU step stays on the CPU
                else:
                    assert v == w, k
        assert all(p.grad is None for p in m.parameters())


def test_restore_to_empty_optimizer_state():
    m = torch.nn.Linear(4, 4)
    o = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
    w = m.weight.detach().clone()
    snap = _snapshot_training_state(m, o)
    _train(m, o, torch.randn(8, 4), 2)
    _restore_training_state(m, o, snap)
    assert len(o.state) == 0 and torch.equal(m.weight, w)
