"""Host-side logic of the slab-decomposed path on CPU (no GPU): the library's slab partition, the NCCL
unique-id broadcast over torch.distributed, the slab slicing / reassembly bench.py and the tests use,
and the peer-mapping exchange of the fused ghost / transpose path, exercised by world_size-2 gloo
process groups."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_1608_03630_b200 import dist as D
        from paper_1608_03630_b200.diffreg import Config, dr_slab
        r, w, _ = D.env_rank_world()
        assert (r, w) == (rank, world)
        cfg = Config(n=(16, 8, 32), nt=2)
        # 1. the unique id rank 0 draws arrives bit-identical everywhere (random bytes stand in for
        #    ncclGetUniqueId, which needs no GPU but may need a network interface)
        uid = os.urandom(128) if rank == 0 else None
        got = D.broadcast_uid(uid, rank)
        ref = [None] * world
        dist.all_gather_object(ref, got)
        assert all(x == ref[0] for x in ref)
        # 2. the slabs tile [0, N3) in rank order, and slicing + gathering a field reproduces it
        z0, nz = dr_slab(cfg, world, rank)
        spans = [None] * world
        dist.all_gather_object(spans, (z0, nz))
        assert spans[0][0] == 0 and all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        assert spans[-1][0] + spans[-1][1] == 32 and len({s[1] for s in spans}) == 1
        v = synth.smooth_vec(3, (16, 8, 32), kmax=3)
        mine = D.slab_of(v, cfg, world, rank)
        assert mine.shape == (3, nz, 8, 16) and mine.is_contiguous()
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        assert torch.equal(D.assemble(parts), v)
        # 3. peer mapping for the fused ghost exchange / transposes (dr_peer_export / dr_peer_import):
        #    every rank receives every rank's (handle, offset) in rank order (a stub context stands in
        #    for the CUDA IPC calls)
        class Stub:
            nranks = world

            def peer_export(self):
                return bytes([rank]) * 64, 4096 * (rank + 1)

            def peer_import(self, handles, offsets):
                self.got = (handles, offsets)

        st = Stub()
        D.map_peers(st)
        assert st.got == ([bytes([r]) * 64 for r in range(world)], [4096 * (r + 1) for r in range(world)])
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_plumbing_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


def test_slab_partition_and_limits():
    from paper_1608_03630_b200 import build
    build.build()
    from paper_1608_03630_b200.diffreg import Config, DiffRegError, dr_slab, dr_workspace_bytes_dist
    cfg = Config(n=(32, 16, 64), nt=4)
    for P in (1, 2, 4, 8):
        spans = [dr_slab(cfg, P, r) for r in range(P)]
        assert [s[0] for s in spans] == [r * 64 // P for r in range(P)] and all(s[1] == 64 // P for s in spans)
        assert dr_workspace_bytes_dist(cfg, P) > 0
    # per-rank workspace shrinks with P (ghost planes and transpose buffers included)
    assert dr_workspace_bytes_dist(cfg, 4) < dr_workspace_bytes_dist(cfg, 2) < dr_workspace_bytes_dist(cfg, 1) * 1.1
    # P must divide N3 and N2, and a slab must hold the 5 upper ghost planes
    assert dr_workspace_bytes_dist(cfg, 3) == 0
    assert dr_workspace_bytes_dist(cfg, 32) == 0          # P does not divide N2 = 16
    assert dr_workspace_bytes_dist(Config(n=(32, 64, 16)), 4) == 0  # N3/P = 4 < 5 ghost planes
    with pytest.raises(DiffRegError):
        dr_slab(cfg, 2, 2)
    # widened ghosts must fit in a slab
    assert dr_workspace_bytes_dist(Config(n=(32, 16, 64), ghost_lo=7, ghost_hi=8), 8) > 0
    assert dr_workspace_bytes_dist(Config(n=(32, 16, 64), ghost_lo=8, ghost_hi=9), 8) == 0
    # too-thin ghosts: a stencil reaches one plane below and two above its cell
    assert dr_workspace_bytes_dist(Config(n=(32, 16, 64), ghost_lo=1, ghost_hi=1), 2) == 0
    assert dr_workspace_bytes_dist(Config(n=(32, 16, 64), ghost_lo=1, ghost_hi=2), 2) > 0
