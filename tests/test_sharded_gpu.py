"""The sharded product path executed on one GPU.

* Row slabs: ``GpuDenseProvider(rows=(b, e))`` (ntf_tensor_upload_rows) holds
  one rank's mode-1 slab (row0 != 0) on a 1-GPU context. Its MTTKRPs are the
  slab's contribution -- the rows of mode 1, the partial sums of the other
  modes -- computed by the same kernels a rank of a multi-GPU run launches
  (fast TMA kernel with the slab's row offset in its unit table, generic
  kernel, dimension-tree partial passes and contractions). Summed over a row
  partition they must equal the oracle's full MTTKRP (kernels.cpp:161-191) at
  the FP64 bar (1e-12).
* One-rank NCCL world: ``Context(nccl_id=...)`` with world 1 creates a real
  communicator, so the drivers take the collective path -- ncclAllGather +
  row compaction for mode 1, ncclAllReduce for the others, the all-reduced
  time budget -- inside the captured CUDA graph. Traces must match the
  oracle like the plain path's.
"""
import numpy as np
import pytest

from parity import compare_traces, rel_fro

pytestmark = pytest.mark.gpu

SHAPES = [
    ([30, 20, 16], 8, [0, 11, 30]),            # generic kernels (small)
    ([64, 48, 40], 20, [0, 21, 43, 64]),       # fast TMA/DMMA kernels, 3 slabs
    ([12, 10, 9, 8], 4, [0, 5, 12]),           # 4-way, split tree
    ([40, 36, 34, 32], 8, [0, 13, 26, 40]),    # 4-way on the fast kernels
]


@pytest.mark.parametrize("flags", [0, 8, 4], ids=["tree", "direct", "generic"])
@pytest.mark.parametrize("shape,rank,cuts", SHAPES, ids=["3way-small", "3way-fast", "4way-small", "4way-fast"])
def test_row_slabs_sum_to_full_mttkrp(P, oracle, shape, rank, cuts, flags):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=77)
    t, _ = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(77, 1))
    want = [oracle.mttkrp(t, init.factors, m) for m in range(len(shape))]
    total = [np.zeros_like(w) for w in want]
    for b, e in zip(cuts[:-1], cuts[1:]):
        prov = P.GpuDenseProvider(np.ascontiguousarray(t[b:e]), full_shape=shape, rows=(b, e))
        got = prov.mttkrp_all(init, flags=flags)
        # mode 1: exactly the slab's rows (the rest zero)
        assert not got[0][:b].any() and not got[0][e:].any()
        for m in range(len(shape)):
            total[m] += got[m]
        # the per-call entry point agrees with the all-modes one on the slab
        for m in range(len(shape)):
            assert rel_fro(prov.mttkrp(init, m), got[m]) <= 1e-12
        prov.close()
    for m in range(len(shape)):
        assert rel_fro(total[m], want[m]) <= 1e-12, (m, rel_fro(total[m], want[m]))


def test_row_slab_rejects_driver_runs(P):
    spec = P.SyntheticSpec(shape=[10, 8, 6], rank=3, noise_sigma=0.0, seed=5)
    t, _ = P.generate(spec)
    init = P.random_init([10, 8, 6], 3, 9)
    prov = P.GpuDenseProvider(np.ascontiguousarray(t[2:7]), full_shape=[10, 8, 6], rows=(2, 7))
    with pytest.raises(P.InvalidArgument):
        P.her_run(prov, init, P.AoConfig(max_outer_iters=2), P.HerParams())
    prov.close()


@pytest.mark.parametrize("shape,rank,sigma,seed", [([64, 48, 40], 20, 0.01, 31), ([20, 18, 16, 14], 5, 0.01, 32),
                                                   ([50, 50, 50], 10, 0.01, 101)])
def test_one_rank_nccl_world_matches_oracle(P, oracle, shape, rank, sigma, seed):
    ctx = P.Context(0, 0, 1, P.Context.nccl_unique_id())
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, seed=seed)
    t, truth = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(seed, 1))
    prov = P.GpuDenseProvider(t, ctx)
    assert abs(prov.norm_sq() - oracle.norm_sq(t)) <= 1e-13 * oracle.norm_sq(t)
    for m in range(len(shape)):  # the per-call provider through allgather / allreduce
        assert rel_fro(prov.mttkrp(init, m), oracle.mttkrp(t, init.factors, m)) <= 1e-12
    model, trace = P.her_run(prov, init, P.AoConfig(max_outer_iters=30), P.HerParams(), ctx=ctx)
    fo, f0, recs = oracle.run("her", t, init.factors, max_outer_iters=30)
    compare_traces(trace, f0, recs, oracle.norm_sq(t), n_check=30)
    # a time budget on a communicator is decided collectively (max-allreduced elapsed time)
    _, tt = P.ao_run(prov, init, P.AoConfig(max_time_s=0.05), ctx=ctx)
    assert len(tt.records) >= 1
    assert tt.records[-1].time_s >= 0.05
    assert all(r.time_s < 0.05 for r in tt.records[:-1])
    prov.close()
    ctx.close()
