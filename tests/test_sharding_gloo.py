"""CPU, world_size 2 over gloo: the multi-GPU choreography of one ESCA iteration.

The engine shards documents across ranks and exchanges only in the M-step
(engine.cu exchange / mstep.cu sparsify + gather_add): each rank
lists its partial C_wk's non-zeros per word row (entries topic | count << 16,
counts above 65535 split into several entries) with an {offset, n} index; the
reduce-scatter adds the other ranks' entries of the own word slice; the reduced
slice is listed the same way; the all-gather adds every other slice's entries
into the (cleared) other rows; every rank then holds the full reduced C_wk and
computes phi / L4 / Q over all rows.  This test runs exactly that choreography on
2 CPU processes with gloo (all_gather_object standing in for the peer-memory
reads), using the product's own host rules (slda_shard_bounds, slda_word_slice
through the C-ABI) and the C oracle for the per-token math, and checks that the
result is bit-identical to the single-process oracle (hence to the reference).
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


def sparsify(Bm, lo, hi):
    """mstep.cu sparsify_kernel: rows [lo, hi) -> ({offset, n} per row, u32 entries)."""
    info, ent = [], []
    for v in range(lo, hi):
        start = len(ent)
        for k in np.nonzero(Bm[v])[0]:
            left = int(Bm[v, k])
            while left:
                piece = min(left, 65535)
                ent.append(int(k) | (piece << 16))
                left -= piece
        info.append((start, len(ent) - start))
    return info, ent


def gather_add(Bm, lst, base, rows):
    """mstep.cu gather_add_kernel for one source list."""
    info, ent = lst
    for v in rows:
        off, n = info[v - base]
        for x in ent[off:off + n]:
            Bm[v, x & 0xFFFF] += x >> 16


def test_sparse_entries_split_large_counts():
    Bm = np.zeros((3, 4), np.int64)
    Bm[1, 2] = 200_000
    Bm[2, 0] = 65535
    info, ent = sparsify(Bm, 0, 3)
    assert info == [(0, 0), (0, 4), (4, 1)]
    back = np.zeros_like(Bm)
    gather_add(back, (info, ent), 0, range(3))
    assert np.array_equal(back, Bm)


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

    rows_per_slice = vpad // world

    def m_step(topic):
        Bl = np.zeros((vpad, K), np.int64)  # this rank's partial C_wk
        np.add.at(Bl, (word[mine], topic), 1)
        # partial list over all rows [0, V): index v - 0
        info1, ent1 = sparsify(Bl, 0, V)
        lists = [None] * world
        dist.all_gather_object(lists, (info1, ent1))
        # reduce-scatter: own slice += the other ranks' entries of it
        for p in range(world):
            if p != rank:
                gather_add(Bl, lists[p], 0, range(r0, r1))
        info2, ent2 = sparsify(Bl, r0, r1)
        Bl[:r0] = 0
        Bl[r1:] = 0
        slices = [None] * world
        dist.all_gather_object(slices, (info2, ent2))
        # all-gather: row v of another slice from its owner v // rows_per_slice, index v - base
        for v in range(V):
            owner = v // rows_per_slice
            if owner != rank:
                gather_add(Bl, slices[owner], owner * rows_per_slice, [v])
        B = Bl[:V]
        # every rank: phi / L4 / Q over all rows
        colsum = B.sum(axis=0)
        denom = colsum.astype(np.float64) + np.float64(V) * BETA
        bhat = ((B.astype(np.float64) + BETA) / denom).astype(np.float32)
        l4 = np.zeros_like(bhat)
        q = np.zeros(V, np.float32)
        for v in range(V):
            out = np.zeros(K, np.float32)
            total = lib.orc_row_prefix(np.ascontiguousarray(bhat[v]), K, out)
            l4[v] = out
            q[v] = falpha * np.float32(total)
        return bhat, l4, q, B.copy()

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
