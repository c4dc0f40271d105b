"""Multi-rank host logic on CPU (gloo, world_size 2): the GPU path shards cells
with no data-path collective, so sharded results must equal the unsharded
ones exactly, and the timed region is reduced with MAX."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1604_05872_b200 import fe, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import port as oracle_port

    cfg = fe.CONFIGS["c2"].with_N(2)
    coords, coeffs, first = shard.shard_inputs(cfg, rank, world, mode)
    A = oracle_port.assemble(cfg, fe.tables(cfg), coords, coeffs)
    t = shard.max_over_ranks(float(rank + 1))
    np.save(os.path.join(out_dir, f"{mode}_{rank}.npy"), A)
    with open(os.path.join(out_dir, f"{mode}_{rank}.txt"), "w") as f:
        f.write(f"{first} {t}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["strong", "weak"])
def test_two_rank_sharding(tmp_path, mode):
    import port as oracle_port

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), mode, str(tmp_path)), nprocs=world, join=True)
    cfg = fe.CONFIGS["c2"].with_N(2)
    parts = [np.load(tmp_path / f"{mode}_{r}.npy") for r in range(world)]
    meta = [open(tmp_path / f"{mode}_{r}.txt").read().split() for r in range(world)]
    assert all(float(m[1]) == 2.0 for m in meta)  # MAX over ranks
    tabs = fe.tables(cfg)
    if mode == "strong":
        coords, coeffs = fe.cell_inputs(cfg)
        full = oracle_port.assemble(cfg, tabs, coords, coeffs)
        assert [int(m[0]) for m in meta] == [0, coords.shape[0] // 2]
        assert np.array_equal(np.concatenate(parts), full)
    else:
        for r in range(world):
            coords, coeffs = fe.cell_inputs(cfg, shard=r)
            assert np.array_equal(parts[r], oracle_port.assemble(cfg, tabs, coords, coeffs))
        assert not np.array_equal(parts[0], parts[1])


def test_cell_range_partition():
    for E in (1, 7, 663552):
        for W in (1, 2, 3, 8):
            ranges = [shard.cell_range(E, r, W) for r in range(W)]
            assert ranges[0][0] == 0 and ranges[-1][1] == E
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.cell_range(10, 2, 2)
