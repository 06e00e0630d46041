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

With the dimension tree (NTF_RUN_DIMTREE) each rank contracts its slab with
A_{N-1} first (Y_slab = T_slab x_{N-1} A_{N-1}, kernels_tree.cu) and forms
blocks 0..N-2 from Y_slab; the exchange is the same (mode 1 gathered, the
others all-reduced), so the same equality must hold.
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


def _slab_tree_mttkrp(t_slab, model, row0, mode):
    """Block `mode` (< N-1) of one slab through Y_slab = T_slab x_{N-1} A_{N-1}."""
    n = t_slab.ndim
    local = [a for a in model]
    local[0] = model[0][row0:row0 + t_slab.shape[0]]
    y = np.tensordot(t_slab, local[n - 1], axes=([n - 1], [0]))  # (I_0..I_{N-2}, r)
    letters = "abcdefg"[: n - 1]
    ops = [y]
    subs = [letters + "z"]
    for j in range(n - 1):
        if j != mode:
            ops.append(local[j])
            subs.append(letters[j] + "z")
    return np.einsum(",".join(subs) + "->" + letters[mode] + "z", *ops)


def _worker(rank, world, port, shape, rank_r, q, tree=False):
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
            if tree and mode < len(shape) - 1:
                part = _slab_tree_mttkrp(slab, model, b, mode)
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


@pytest.mark.parametrize("tree", [False, True], ids=["direct", "dimtree"])
@pytest.mark.parametrize("shape", [[7, 6, 5], [9, 4, 3, 5]])
def test_slab_sharded_mttkrp_world2(shape, tree):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + len(shape) + (10 if tree else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, 3, q, tree)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(2):
        assert max(results[rank]) < 1e-12, results[rank]
