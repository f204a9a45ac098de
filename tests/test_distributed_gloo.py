"""World-size-2 (and 3) gloo runs of DistributedDomain on CPU.

The CUDA engines and the device halo are replaced by the oracle engine and
a protocol-level halo (read_slots / write_slots + gloo isend/irecv), so this
exercises exactly the host-side multi-rank logic of the N > 1 path: block
assignment (reference balance), half-plans on each rank, the per-peer
message schedule (one message per peer per phase, edge order), and both
drivers — and checks the gathered result against the reference's
single-process golden bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import flags_of, golden_files, load_golden, params_of, stencil_of

DOMAIN = {os.path.basename(p)[:-4]: p for p in golden_files("domain")}


class ProtocolHalo:
    """Test stand-in for DeviceHalo: moves values with the engine protocol."""

    def __init__(self, device, world=1):
        self.world = world
        self.local = {0: [], 1: []}
        self.sends = {0: {}, 1: {}}
        self.recvs = {0: {}, 1: {}}

    def add_local(self, phase, src, dst, pp):
        self.local[phase.value].append((src, dst, pp.send_sel, pp.take, pp.tgt_sel))

    def add_send(self, phase, src, peer, pp):
        self.sends[phase.value].setdefault(peer, []).append((src, pp.send_sel))

    def add_recv(self, phase, dst, peer, pp):
        self.recvs[phase.value].setdefault(peer, []).append(
            (dst, pp.n_msg, pp.take, pp.tgt_sel))

    def commit(self, comm=None):
        pass

    def start(self, phase, stream):
        import torch
        import torch.distributed as dist

        ph = phase.value
        staged = [(dst, src.read_slots(send)[take], tgt) for src, dst, send, take, tgt in self.local[ph]]
        reqs, inbox = [], {}
        for peer, lst in sorted(self.sends[ph].items()):
            msg = np.concatenate([src.read_slots(sel) for src, sel in lst])
            reqs.append(dist.isend(torch.from_numpy(msg), dst=peer))
        for peer, lst in sorted(self.recvs[ph].items()):
            buf = torch.empty(sum(n for _, n, _, _ in lst), dtype=torch.float64)
            inbox[peer] = buf
            reqs.append(dist.irecv(buf, src=peer))
        for r in reqs:
            r.wait()
        for dst, vals, tgt in staged:
            dst.write_slots(tgt, vals)
        for peer, lst in sorted(self.recvs[ph].items()):
            msg = inbox[peer].numpy()
            off = 0
            for dst, n, take, tgt in lst:
                dst.write_slots(tgt, msg[off:off + n][take])
                off += n

    def wait(self, stream):
        pass


def _oracle_engine(flags, stencil, params, pattern, frame_width, device, kind="sparse"):
    from oracle.sparse_ref import OracleSparseEngine

    return OracleSparseEngine(flags, stencil, params, pattern, frame_width=frame_width)


def _worker(rank, world, port, path, pattern, driver, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_06880_b200.domain import DistributedDomain

    rec = load_golden(path)
    dom = DistributedDomain(flags_of(rec), tuple(int(b) for b in rec["block"]), stencil_of(rec),
                            params_of(rec), pattern=pattern, frame_width=1, rank=rank, world=world,
                            device=0, engine_factory=_oracle_engine,
                            halo_factory=lambda dev: ProtocolHalo(dev, world))
    dom.init_random(int(rec["seed"]))
    dom.run(int(rec["steps"]), driver=driver)
    full = dom.gather_canonical_global()
    ranks_used = sorted(set(dom.assignment.values()))
    if rank == 0:
        np.save(os.path.join(out_dir, "full.npy"), full)
        np.save(os.path.join(out_dir, "ranks.npy"), np.array(ranks_used))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world,pattern,driver", [
    ("domain_d3q19_2x2x2", 2, "aa", "overlapped"),
    ("domain_d3q19_2x2x2", 3, "pull", "sequential"),
    ("domain_d2q9_riverbed", 2, "aa", "sequential"),
    ("domain_d3q27_riverbed", 2, "pull", "overlapped"),
])
def test_gloo_multi_rank_matches_single_process_golden(name, world, pattern, driver, tmp_path):
    path = DOMAIN[name]
    mp.start_processes(_worker, args=(world, _free_port(), path, pattern, driver, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    rec = load_golden(path)
    full = np.load(tmp_path / "full.npy")
    assert list(np.load(tmp_path / "ranks.npy")) == list(range(world))
    np.testing.assert_array_equal(full, rec[f"{pattern}_final"])
