"""he_train's chunk pipeline (host logic, CPU): chunks keep the sample order,
the last chunk may be short, and each chunk's H2D is staged before the
previous chunk is handed out for compute."""

from paper_2403_20190_b200 import hewnn


def test_chunks_staged_order(monkeypatch):
    events = []

    class FakeStaged:
        def __init__(self, samples):
            events.append(("stage", tuple(samples)))

    monkeypatch.setattr(hewnn, "_Staged", FakeStaged)
    seen = []
    for chunk, staged in hewnn._chunks_staged(iter(range(7)), 3, check=seen.append):
        events.append(("run", tuple(chunk)))
        assert isinstance(staged, FakeStaged)
    assert seen == list(range(7))
    assert events == [("stage", (0, 1, 2)), ("stage", (3, 4, 5)), ("run", (0, 1, 2)),
                      ("stage", (6,)), ("run", (3, 4, 5)), ("run", (6,))]


def test_chunks_staged_empty_and_exact(monkeypatch):
    monkeypatch.setattr(hewnn, "_Staged", lambda s: None)
    assert list(hewnn._chunks_staged(iter([]), 4)) == []
    out = [tuple(c) for c, _ in hewnn._chunks_staged(iter(range(8)), 4)]
    assert out == [(0, 1, 2, 3), (4, 5, 6, 7)]
