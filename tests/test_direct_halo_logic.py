"""Host-side logic of direct local halo edges (CPU): a model of one local
edge -- source slot s of block B, ghost slot g of block A -- stepped by the
copy program (CANONICAL g <- s before the even step, REVERSED s <- g before
the odd step) and by a linked group (the even step reads and writes s
directly) driven through Domain.run / step calls with the call-boundary
handling of Domain._stale_before / _stale_after and CUDA-graph pairs
replayed by key.  After every call both models must hold the same (s, g)."""

import random

from paper_2408_06880_b200.domain import Domain


class _Group:
    def __init__(self, model):
        self.model = model

    def stale_copy(self, mode, stream):
        self.model.issue(("stale", mode))


class _Linked(Domain):
    """Domain with the device replaced by the slot model: kernels are ops
    ("sweep", parity) / ("stale", mode) applied to the two slots; a CUDA
    graph is the op list its capture issued, replayed by the same key as
    Domain._replay_pair."""

    def __init__(self):  # noqa: D401 - no engines, no device
        self.direct_halo = True
        self._left = 1
        self._stale_pending = False
        self._stream = 0
        self.check = "deferred"
        self.steps_done = 0
        self.par = 0
        self.k = 0
        self.slots = {"s": ("init",), "g": ("ghost0",)}
        self.recording = None
        self._group = _Group(self)
        self.graphs = {}

    @property
    def parity(self):
        return self.par

    def _graph_capable(self):
        return True

    def _driver(self, name):
        return self._step

    def issue(self, op):
        if self.recording is not None:
            self.recording.append(op)
        self.apply(op)

    def apply(self, op):
        sl = self.slots
        if op[0] == "stale":
            if op[1] == 0:
                sl["g"] = sl["s"]
            elif op[1] == 1:
                sl["s"], sl["g"] = sl["g"], sl["s"]
            else:
                sl["s"] = sl["g"]
        else:  # the sweep: the combined step (E) or the cell-local step (O)
            sl["s"] = ("E" if op[1] == 0 else "O", self.k, sl["s"])

    def _step(self):
        self._stale_before()
        self.issue(("sweep", self.par))
        self._stale_after()
        self.par ^= 1
        self.k += 1

    def _replay_pair(self, driver, fn):
        key = (driver, self.par, (), self.direct_halo and self._left == 2)
        if key not in self.graphs:  # capture runs the pair once, recording
            self.recording = []
            fn()
            fn()
            self.graphs[key] = self.recording
            self.recording = None
            return
        for op in self.graphs[key]:  # replay: the captured ops, same order
            self.apply(op)
            if op[0] == "sweep":
                self.k += 1
                self.par ^= 1


class _Copy:
    def __init__(self):
        self.par, self.k = 0, 0
        self.slots = {"s": ("init",), "g": ("ghost0",)}

    def run(self, n):
        for _ in range(n):
            if self.par == 0:
                self.slots["g"] = self.slots["s"]  # CANONICAL
                self.slots["g"] = ("E", self.k, self.slots["g"])
            else:
                self.slots["s"] = self.slots["g"]  # REVERSED
                self.slots["s"] = ("O", self.k, self.slots["s"])
            self.par ^= 1
            self.k += 1


def test_calls_hand_back_the_copy_programs_state():
    rng = random.Random(7)
    for trial in range(200):
        d, c = _Linked(), _Copy()
        for _ in range(12):
            n = rng.choice([1, 1, 2, 3, 4, 5, 6, 9])
            graph = rng.random() < 0.6
            if rng.random() < 0.2:
                d._step()  # a public single-step call (outside run)
                d.steps_done += 1
                c.run(1)
            else:
                d.run(n, use_graph=graph)
                c.run(n)
            assert d.slots == c.slots, (trial, n, graph, d.slots, c.slots)
            assert d.par == c.par and d.k == c.k
