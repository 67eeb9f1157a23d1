"""Multi-rank host logic on CPU: world_size 2 over gloo.

* the NCCL unique-id broadcast used by dist.init_distributed();
* the all-gather of the NVLink peer-exchange IPC handles
  (dist.open_peer_exchange);
* the row-sharded GK arithmetic (tests/sharded_model.py, the same data
  movement as the CUDA path at N GPUs) against the single-process oracle:
  alphas/betas, k', the gathered left basis and the rank count.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import krylov_oracle as O
        from paper_2104_10785_b200 import _lib
        from paper_2104_10785_b200.dist import broadcast_uid
        from paper_2104_10785_b200.synth import low_rank_synth
        from tests.sharded_model import allreduce, sharded_gk

        out = {}
        uid = _lib.nccl_unique_id() if rank == 0 else None
        got = broadcast_uid(uid, rank)
        out["uid"] = got

        # peer-exchange plumbing: every rank's IPC handle reaches every rank
        # in rank order (the context is mocked: no GPU here)
        from paper_2104_10785_b200.dist import open_peer_exchange

        class _MockCtx:
            nranks = world

            def __init__(self):
                self.rank, self.slot, self.handles = rank, None, None

            def px_export(self, slot):
                self.slot = slot
                return bytes([17 * (rank + 1)]) * _lib.PX_HANDLE_BYTES

            def px_open(self, handles):
                self.handles = handles
                return True

        mctx = _MockCtx()
        out["px"] = (open_peer_exchange(mctx, slot=4096), mctx.slot, mctx.handles)
        cases = [(301, 120, 25, 60, 3), (1000, 400, 100, 400, 5), (257, 200, 200, 200, 11)]
        res = []
        for m, n, l, k, seed in cases:
            A = low_rank_synth(m, n, l, seed=seed)
            g = sharded_gk(A, k, seed=seed)
            Qfull = np.zeros((m, g["Q"].shape[1]))
            Qfull[g["row0"]:g["row0"] + g["Q"].shape[0]] = g["Q"]
            Qfull = allreduce(Qfull)  # gather the row shards
            res.append((g["alphas"], g["betas"], g["k_prime"], Qfull, g["P"]))
        out["res"] = res
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharded_gk_matches_oracle():
    from oracle import krylov_oracle as O
    from paper_2104_10785_b200.synth import low_rank_synth
    from tests.parity import assert_gk_match

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank received rank 0's NCCL id
    assert outs[0]["uid"] == outs[1]["uid"] and len(outs[0]["uid"]) == 128
    # ... and every rank's peer-exchange handle, in rank order
    want = b"".join(bytes([17 * (r + 1)]) * 64 for r in range(world))
    for r in range(world):
        assert outs[r]["px"] == (True, 4096, want)
    cases = [(301, 120, 25, 60, 3), (1000, 400, 100, 400, 5), (257, 200, 200, 200, 11)]
    for ci, (m, n, l, k, seed) in enumerate(cases):
        A = low_rank_synth(m, n, l, seed=seed)
        ref = O.gk_oracle(A, k, seed=seed)
        for r in range(world):
            a, b, kp, Qf, P = outs[r]["res"][ci]
            # both ranks agree bit for bit on the replicated quantities
            assert np.array_equal(a, outs[0]["res"][ci][0])
            assert np.array_equal(P, outs[0]["res"][ci][4])
            assert_gk_match(a, b, kp, ref.alphas, ref.betas, ref.k_prime, what=str(ci))
            ncol = min(Qf.shape[1], ref.Q.shape[1], kp, 8)
            cos = np.abs(np.einsum("ij,ij->j", Qf[:, :ncol], ref.Q[:, :ncol]))
            assert cos.min() >= 1 - 1e-8
        # rank count from the sharded scalars equals the oracle's
        th, _ = O.ql_eig(*O.gram_of(outs[0]["res"][ci][0], outs[0]["res"][ci][1][:kp + 1]),
                         vectors=False)
        th_ref, _ = O.ql_eig(*O.gram_of(ref.alphas, ref.betas), vectors=False)
        assert O.threshold_count(th, 1e-8, "absolute")[0] == \
            O.threshold_count(th_ref, 1e-8, "absolute")[0]
