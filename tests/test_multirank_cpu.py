"""World-size-2 CPU (gloo) check of the mode-1 slab sharding the multi-GPU
path uses.

Each rank holds the rows [begin, end) of mode 1 that ``slab_range`` (the
product's own C-ABI host function) assigns it. Per mode:
  * mode 1: the rank computes its slab's MTTKRP rows, the rows are exchanged
    with a padded all-gather and compacted in rank order (the NCCL
    ncclAllGather + compact_rows_kernel sequence of MttkrpEngine::run);
  * modes != 1: the rank contracts its slab into a partial I_n x r MTTKRP and
    the partials are summed with an all-reduce (ncclAllReduce).
The result must equal the single-process MTTKRP of the full tensor, and
||T||^2 must equal the all-reduced slab norms. The algebra is evaluated with
the oracle (test infrastructure) on each slab; the collectives are gloo.

With the dimension tree (NTF_RUN_DIMTREE, split h) each rank contracts its
slab into Y_L = T_slab x_h A_h .. x_{N-1} A_{N-1} (local rows) and
Y_R = T_slab x_0 A_0 .. x_{h-1} A_{h-1} (a partial sum over the slab) and
forms the blocks from them (kernels_tree.cu); the exchange is the same
(mode 1 gathered, the others all-reduced, by linearity in Y_R), so the same
equality must hold for every split.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _slab_mttkrp(oracle, t_slab, model, row0, mode):
    """MTTKRP of one mode-1 slab with the slab's rows of A_1."""
    local = [a.copy() for a in model]
    local[0] = model[0][row0:row0 + t_slab.shape[0]]
    return oracle.mttkrp(t_slab, local, mode)


def _slab_tree_mttkrp(t_slab, model, row0, mode, split):
    """Block `mode` of one slab through the split dimension tree (runtime.cpp
    MttkrpEngine): blocks < h contract Y_L = T_slab x_h A_h .. x_{N-1} A_{N-1},
    blocks >= h contract Y_R = T_slab x_0 A_0(slab rows) .. x_{h-1} A_{h-1};
    with h = N-1, block N-1 is the direct slab MTTKRP."""
    n = t_slab.ndim
    local = [a for a in model]
    local[0] = model[0][row0:row0 + t_slab.shape[0]]
    letters = "abcdefg"[:n]
    lo, hi = (0, split) if mode < split else (split, n)
    # contract the other side of the split first
    ops, subs = [t_slab], [letters]
    for j in range(n):
        if not lo <= j < hi:
            ops.append(local[j])
            subs.append(letters[j] + "z")
    y = np.einsum(",".join(subs) + "->" + letters[lo:hi] + "z", *ops)
    ops, subs = [y], [letters[lo:hi] + "z"]
    for j in range(lo, hi):
        if j != mode:
            ops.append(local[j])
            subs.append(letters[j] + "z")
    return np.einsum(",".join(subs) + "->" + letters[mode] + "z", *ops)


def _worker(rank, world, port, shape, rank_r, q, split=0):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2001_04321_b200 as P
        import pyoracle as O
        t, _ = O.generate(shape, rank_r, sigma=0.05, seed=77)
        model = O.random_init(shape, rank_r, 78)
        b, e = P.slab_range(shape[0], rank, world)
        slab = np.ascontiguousarray(t[b:e])
        nsq = torch.tensor([O.norm_sq(slab)], dtype=torch.float64)
        dist.all_reduce(nsq)
        errs = [abs(nsq.item() - O.norm_sq(t)) / O.norm_sq(t)]
        maxrows = max(P.slab_range(shape[0], p, world)[1] - P.slab_range(shape[0], p, world)[0]
                      for p in range(world))
        for mode in range(len(shape)):
            if split:
                part = _slab_tree_mttkrp(slab, model, b, mode, split)
            else:
                part = _slab_mttkrp(O, slab, model, b, mode)
            if mode == 0:
                pad = torch.zeros(maxrows, rank_r, dtype=torch.float64)
                pad[: e - b] = torch.from_numpy(part)
                bufs = [torch.zeros_like(pad) for _ in range(world)]
                dist.all_gather(bufs, pad)
                full = np.concatenate([bufs[p][: P.slab_range(shape[0], p, world)[1]
                                                - P.slab_range(shape[0], p, world)[0]].numpy()
                                       for p in range(world)])
            else:
                red = torch.from_numpy(part.copy())
                dist.all_reduce(red)
                full = red.numpy()
            want = O.mttkrp(t, model, mode)
            errs.append(float(np.linalg.norm(full - want) / np.linalg.norm(want)))
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split", [0, 1, 2, 3], ids=["direct", "tree-h1", "tree-h2", "tree-h3"])
@pytest.mark.parametrize("shape", [[7, 6, 5], [9, 4, 3, 5]])
def test_slab_sharded_mttkrp_world2(shape, split):
    if split >= len(shape):
        pytest.skip("split must be < N")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + len(shape) + 10 * split
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, 3, q, split)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(2):
        assert max(results[rank]) < 1e-12, results[rank]
