"""CPU, world_size 2 over gloo: the multi-GPU choreography of one ESCA iteration.

The engine shards documents across ranks and exchanges only in the M-step
(engine.cu m_step): reduce-scatter of C_wk by word-row slices,
all-reduce of the column sums C_k, phi/L4/Q on the own slice, all-gather.
This test runs exactly that choreography on 2 CPU processes with gloo, using
the product's own host rules (slda_shard_bounds, slda_word_slice through the
C-ABI) and the C oracle for the per-token math, and checks that the result is
bit-identical to the single-process oracle (hence to the reference).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import abi
from oracle_lib import OracleModel, digest, oracle_lib, random_corpus

D, V, K, SEED, ITERS = 80, 37, 8, 1234, 3
BETA = 0.01


def _corpus():
    return random_corpus(D, V, 20.0, 77)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = oracle_lib()
    doc, word = _corpus()
    T = len(doc)
    alpha = 50.0 / K
    falpha = np.float32(alpha)
    lens = np.bincount(doc, minlength=D).astype(np.uint32)
    bounds = np.zeros(world + 1, np.uint32)
    abi.check(abi.lib().slda_shard_bounds(D, T, lens.ctypes.data, world, bounds.ctypes.data))
    b, e = int(bounds[rank]), int(bounds[rank + 1])
    r0, r1, vpad = C.c_uint32(), C.c_uint32(), C.c_uint32()
    abi.check(abi.lib().slda_word_slice(V, world, rank, C.byref(r0), C.byref(r1), C.byref(vpad)))
    r0, r1, vpad = r0.value, r1.value, vpad.value
    mine = np.nonzero((doc >= b) & (doc < e))[0]  # corpus positions == RNG element ids
    # trainer.cpp:383-388: uniform initial topics keyed by corpus position
    topic = np.array([lib.orc_uniform_topic(SEED, 0xFFFFFFFF, int(t), K) for t in mine], np.uint32)

    def m_step(topic):
        # local C_wk, then reduce-scatter by word rows (gloo: all_reduce + own slice)
        Bl = np.zeros((vpad, K), np.int64)
        np.add.at(Bl, (word[mine], topic), 1)
        Bt = torch.from_numpy(Bl)
        dist.all_reduce(Bt)
        Bs = Bt.numpy()[r0:r1]
        colsum = torch.from_numpy(Bs.sum(axis=0).astype(np.int64))
        dist.all_reduce(colsum)  # C_k
        denom = colsum.numpy().astype(np.float64) + np.float64(V) * BETA
        bhat_s = ((Bs.astype(np.float64) + BETA) / denom).astype(np.float32)
        l4_s = np.zeros_like(bhat_s)
        q_s = np.zeros(r1 - r0, np.float32)
        for i in range(r1 - r0):
            row = np.ascontiguousarray(bhat_s[i])
            out = np.zeros(K, np.float32)
            total = lib.orc_row_prefix(row, K, out)
            l4_s[i] = out
            q_s[i] = falpha * np.float32(total)
        # all-gather the slices (equal-sized over V_pad rows)
        rows = vpad // world

        def gather(x):
            pad = np.zeros((rows,) + x.shape[1:], x.dtype)
            pad[: len(x)] = x
            parts = [torch.zeros_like(torch.from_numpy(pad)) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(pad))
            return np.concatenate([p.numpy() for p in parts])[:V]

        return gather(bhat_s), gather(l4_s), gather(q_s), gather(Bs.astype(np.int64))

    bhat, l4, q, B = m_step(topic)
    for it in range(ITERS):
        # C_dk rows of the own documents (rebuild_doc_topic), then the E-step.
        rows = {}
        for d in range(b, e):
            t = topic[doc[mine] == d]
            u, c = np.unique(t, return_counts=True)
            rows[d] = (u.astype(np.uint32), c.astype(np.uint32))
        new = np.empty_like(topic)
        u0, u1 = C.c_double(), C.c_double()
        for j, t in enumerate(mine):
            tops, cnts = rows[int(doc[t])]
            w = int(word[t])
            lib.orc_uniform2(SEED, it, int(t), C.byref(u0), C.byref(u1))
            new[j] = lib.orc_sample_token(len(tops), tops, cnts, np.ascontiguousarray(bhat[w]), float(q[w]),
                                          np.ascontiguousarray(l4[w]), K, u0.value, u1.value)
        topic = new
        bhat, l4, q, B = m_step(topic)
    # gather assignments in corpus order
    full = torch.zeros(T, dtype=torch.int64)
    full[torch.from_numpy(mine)] = torch.from_numpy(topic.astype(np.int64))
    dist.all_reduce(full)
    if rank == 0:
        np.savez(os.path.join(out_dir, "sharded.npz"), assignments=full.numpy().astype(np.uint32),
                 bhat=bhat, l4=l4, q=q, B=B.astype(np.uint32))
    dist.destroy_process_group()


def test_two_rank_choreography_is_bit_identical(tmp_path):
    port = _free_port()
    mp.spawn(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "sharded.npz")
    doc, word = _corpus()
    ref = OracleModel(D, V, doc, word, None, K=K, seed=SEED)
    for _ in range(ITERS):
        ref.iterate()
    assert digest(got["assignments"]) == digest(ref.assignments())
    assert digest(got["B"]) == digest(ref.word_topic())
    assert digest(got["bhat"]) == digest(ref.word_topic_prob())
    assert digest(got["l4"]) == digest(ref.l4())
    assert digest(got["q"]) == digest(ref.tree_mass())


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_word_slices_tile_the_vocabulary(world):
    covered = []
    for rank in range(world):
        b, e, p = C.c_uint32(), C.c_uint32(), C.c_uint32()
        abi.check(abi.lib().slda_word_slice(141000, world, rank, C.byref(b), C.byref(e), C.byref(p)))
        assert p.value % world == 0 and p.value >= 141000
        covered.append((b.value, e.value))
    assert covered[0][0] == 0 and covered[-1][1] == 141000
    assert all(covered[i][1] == covered[i + 1][0] for i in range(world - 1))
