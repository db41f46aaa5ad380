"""Host-side logic of the N>1 path on CPU with the gloo backend (world_size 2): NCCL unique-id
broadcast, slab partition of the global z range, and max-over-ranks timing reduction."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C
    import paper_2502_20049_b200 as psm
    nid = [None]
    if rank == 0:
        try:
            nid[0] = psm.psm_nccl_get_unique_id()
        except psm.PSMError:
            nid[0] = bytes(range(128))  # no network interface for NCCL bootstrap: any 128 B
    dist.broadcast_object_list(nid, 0)
    assert len(nid[0]) == 128
    buf = (C.c_uint8 * 128).from_buffer_copy(nid[0])
    nz = 37
    g = psm.psm_grid(24, 20, nz, (C.c_int32 * 3)(0, 0, 0))
    o = psm.psm_options(psm.PSM_F32, psm.PSM_TWO_ARRAY, 1, 1, (C.c_double * 3)(0, 0, 0), rank,
                        world, C.cast(buf, C.c_void_p), None, 0, 0.1875)
    ctx = psm.psm_create(g, 19, 0.6, o)  # host-only: no device touched
    z0, nzl = psm.psm_local_extent(ctx)
    psm.psm_destroy(ctx)
    ext = [None] * world
    dist.all_gather_object(ext, (z0, nzl))
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((ext, float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_partition_and_id_broadcast_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ext, tmax = q.get(timeout=10)
    # slabs tile [0, nz) exactly, in rank order, balanced to within one plane
    zs = 0
    for z0, nzl in ext:
        assert z0 == zs and nzl >= 1
        zs += nzl
    assert zs == 37
    assert max(n for _, n in ext) - min(n for _, n in ext) <= 1
    assert tmax == float(world)
