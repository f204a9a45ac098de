"""Multi-rank paths on one GPU:

* loopback: every halo edge travels as a real NCCL message (ncclSend /
  ncclRecv inside one group on the comm stream) from rank 0 to itself, so
  pack kernel -> NCCL -> unpack kernel is exercised exactly as between GPUs;
* the peer transport (CUDA IPC + epoch flags, no NCCL) in loopback and with
  two processes sharing the GPU through IPC mappings of each other's
  buffers;
* two processes sharing the GPU with the host-staged transport (gloo),
  blocks split between the ranks by the reference's balance.

Both must reproduce the reference's single-process golden bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import flags_of, golden_files, load_golden, params_of, stencil_of

pytestmark = pytest.mark.gpu

DOMAIN = {os.path.basename(p)[:-4]: p for p in golden_files("domain")}


@pytest.mark.parametrize("pattern", ["aa", "pull"])
@pytest.mark.parametrize("name", ["domain_d3q19_2x2x2", "domain_d3q27_riverbed",
                                  "domain_d2q9_riverbed"])
def test_nccl_loopback_matches_golden(name, pattern, gpu_lib):
    from paper_2408_06880_b200.domain import DistributedDomain

    rec = load_golden(DOMAIN[name])
    dom = DistributedDomain(flags_of(rec), tuple(int(b) for b in rec["block"]), stencil_of(rec),
                            params_of(rec), pattern=pattern, frame_width=1, rank=0, world=1,
                            device=0, loopback=True)
    dom.init_random(int(rec["seed"]))
    dom.run(int(rec["steps"]), driver="overlapped")
    np.testing.assert_array_equal(dom.gather_canonical(), rec[f"{pattern}_final"])


@pytest.mark.parametrize("pattern", ["aa", "pull"])
@pytest.mark.parametrize("name", ["domain_d3q19_2x2x2", "domain_d3q27_riverbed"])
def test_peer_loopback_matches_golden(name, pattern, gpu_lib):
    """Peer transport, every edge a message to this rank through its own
    buffers: remote pack -> release flag -> acquire wait -> unpack -> ack."""
    from paper_2408_06880_b200.domain import DistributedDomain

    rec = load_golden(DOMAIN[name])
    for use_graph in (False, True):
        dom = DistributedDomain(flags_of(rec), tuple(int(b) for b in rec["block"]),
                                stencil_of(rec), params_of(rec), pattern=pattern, frame_width=1,
                                rank=0, world=1, device=0, loopback=True, transport="p2p")
        dom.init_random(int(rec["seed"]))
        dom.run(int(rec["steps"]), driver="overlapped", use_graph=use_graph)
        np.testing.assert_array_equal(dom.gather_canonical(), rec[f"{pattern}_final"])


def _worker(rank, world, port, path, pattern, out_dir, transport="host", frame=1):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_06880_b200.domain import DistributedDomain

    rec = load_golden(path)
    dom = DistributedDomain(flags_of(rec), tuple(int(b) for b in rec["block"]), stencil_of(rec),
                            params_of(rec), pattern=pattern, frame_width=frame, rank=rank,
                            world=world, device=0, transport=transport)
    if frame == "halo":
        # per-face frames: only faces towards the other rank's blocks
        local = {b.bid for b in dom.local_blocks()}
        assert dom._face_frames
        assert any(dom.blocks[n].rank == rank for b in dom.local_blocks()
                   for n in b.neighbors.values() if n not in (b.bid,)) or len(local) == 1
    dom.init_random(int(rec["seed"]))
    steps = int(rec["steps"])
    if transport == "p2p":
        # device-side epochs: CUDA-graph replays across processes stay in step
        dom.run(1, driver="overlapped")
        dom.run(steps - 1, driver="overlapped", use_graph=True)
    else:
        dom.run(steps, driver="overlapped")
    full = dom.gather_canonical_global()
    if rank == 0:
        np.save(os.path.join(out_dir, "full.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,pattern", [("domain_d3q19_2x2x2", "aa"),
                                          ("domain_d3q19_walled_strips", "pull")])
def test_two_ranks_host_staged_match_golden(name, pattern, tmp_path, gpu_lib):
    path = DOMAIN[name]
    mp.start_processes(_worker, args=(2, _free_port(), path, pattern, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    rec = load_golden(path)
    np.testing.assert_array_equal(np.load(tmp_path / "full.npy"), rec[f"{pattern}_final"])


@pytest.mark.parametrize("name,pattern", [("domain_d3q19_2x2x2", "aa")])
def test_two_ranks_peer_ipc_match_golden(name, pattern, tmp_path, gpu_lib):
    """Two processes on one GPU, each mapping the other's receive buffer and
    flags through CUDA IPC: the same code path as two GPUs over NVLink."""
    path = DOMAIN[name]
    mp.start_processes(_worker, args=(2, _free_port(), path, pattern, str(tmp_path), "p2p"),
                       nprocs=2, join=True, start_method="spawn")
    rec = load_golden(path)
    np.testing.assert_array_equal(np.load(tmp_path / "full.npy"), rec[f"{pattern}_final"])


@pytest.mark.parametrize("transport", ["host", "p2p"])
@pytest.mark.parametrize("name,pattern", [("domain_d3q19_2x2x2", "aa"),
                                          ("domain_d3q27_riverbed", "pull")])
def test_two_ranks_face_frames_match_golden(name, pattern, transport, tmp_path, gpu_lib):
    """frame_width="halo" with blocks of both ranks interleaved: frames only
    on faces towards remote blocks, local edges ahead of the interior sweep
    on the compute stream, remote ones overlapped — same bits as the
    reference's single-process run."""
    path = DOMAIN[name]
    mp.start_processes(_worker, args=(2, _free_port(), path, pattern, str(tmp_path), transport,
                                      "halo"),
                       nprocs=2, join=True, start_method="spawn")
    rec = load_golden(path)
    np.testing.assert_array_equal(np.load(tmp_path / "full.npy"), rec[f"{pattern}_final"])
