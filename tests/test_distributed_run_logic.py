"""Host logic of DistributedDomain.run (CPU): with the NCCL transport and
more than one rank, the first step pair of a graph run is taken eagerly so
NCCL's lazy peer connection happens outside stream capture; every later call
(and every other transport) goes straight to the graph path."""

from paper_2408_06880_b200 import domain as D


def _calls(monkeypatch, eager_first, runs):
    seen = []
    monkeypatch.setattr(D.Domain, "run",
                        lambda self, steps, driver="sequential", use_graph=False:
                        seen.append((steps, driver, use_graph)))
    dom = object.__new__(D.DistributedDomain)
    dom._eager_first = eager_first
    for steps, use_graph in runs:
        dom.run(steps, use_graph=use_graph)
    return seen


def test_first_graph_run_starts_eagerly(monkeypatch):
    seen = _calls(monkeypatch, True, [(7, True), (4, True)])
    assert seen == [(2, "overlapped", False), (5, "overlapped", True), (4, "overlapped", True)]


def test_single_step_and_eager_runs(monkeypatch):
    # one step: all of it eager; eager runs leave the flag for the first graph run
    assert _calls(monkeypatch, True, [(1, True), (3, True)]) == [
        (1, "overlapped", False), (0, "overlapped", True), (3, "overlapped", True)]
    assert _calls(monkeypatch, True, [(3, False), (2, True)]) == [
        (3, "overlapped", False), (2, "overlapped", False), (0, "overlapped", True)]


def test_other_transports_unchanged(monkeypatch):
    assert _calls(monkeypatch, False, [(6, True)]) == [(6, "overlapped", True)]
