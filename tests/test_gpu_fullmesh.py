"""Parity at the benchmark's execution scale (VERDICT r01 "next" #1).

* Every cell of every full BASELINE mesh, assembled by the exact call bench.py
  times (``femgpu_assemble`` on device-resident cell-major inputs, one launch
  over the whole mesh), against the reference's CPU path -- femopt's optimized
  emitted C on all host threads (oracle/parity.py) -- at 1e-12 relative
  Frobenius error per element.  The reference checks every kernel over its
  whole output the same way (proj/tests/test_backend.cpp:167-182).
* Multi-tile runs: E >= 3 x (persistent grid) x (cells per tile) + an odd
  remainder, so every persistent CTA runs >= 3 tiles and the ring / staging
  handoffs between tiles (double-buffered g tiles, sFull/sEmpty, prologue of
  tile i+1 under the epilogue of tile i, TMA ring wrap) are compared with the
  reference, and also with the C restatement (oracle/femoracle.c).
* Contiguous shards (the multi-GPU partition): launches over
  [lo, hi) slices give the unsharded output bit for bit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1604_05872_b200 import fe, femgpu, shard  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-12
CONFIGS = ["c1", "c2", "c3", "c4", "c5"]

# cells per launch such that every persistent CTA of the config's kernel runs
# >= 3 tiles: c1 444 CTAs x 256-cell stages; c2 148 x 32; c3 296 x 8;
# c4 148 x 16; c5 148 x 16 -- rounded up, plus an odd remainder
MULTI_TILE = {"c1": 3 * 444 * 256 + 77, "c2": 3 * 148 * 32 + 97, "c3": 3 * 296 * 8 + 13,
              "c4": 3 * 148 * 16 + 13, "c5": 3 * 148 * 16 + 13}


def _device_launch(cfg, coords, coeffs, schedule=femgpu.SCHED_AUTO):
    dev = torch.device("cuda:0")
    form = femgpu.Form.from_config(cfg, schedule=schedule)
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    out = torch.full((coords.shape[0], cfg.n, cfg.n), float("nan"), dtype=torch.float64,
                     device=dev)
    form.assemble(x, c, out, stream=torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    return form, out


@pytest.mark.parametrize("name", CONFIGS)
def test_full_mesh_every_cell_vs_reference(name):
    import parity

    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg)
    _, out = _device_launch(cfg, coords, coeffs)
    r = parity.check(cfg, coords, coeffs, lambda a, b: out[a:b].cpu().numpy())
    assert r["cells_checked"] == cfg.ncells
    assert r["max_frob_rel"] < TOL, r


# the second schedule of each family, on the same full meshes (the cost model
# ranks them behind AUTO's choice; profiles/schedule_choice_r02.json)
ALTERNATIVES = [("c2", femgpu.SCHED_QUADRATURE, "helm_quad_kernel"),
                ("c3", femgpu.SCHED_TENSOR, "elas_tensor_kernel"),
                ("c4", femgpu.SCHED_QUADRATURE_MMA, "svk_mma_kernel"),
                ("c5", femgpu.SCHED_QUADRATURE, "burgers_quad_kernel")]


@pytest.mark.parametrize("name,schedule,kernel", ALTERNATIVES)
def test_full_mesh_alternative_schedules_vs_reference(name, schedule, kernel):
    import parity

    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg)
    form, out = _device_launch(cfg, coords, coeffs, schedule)
    assert form.info["kernel_name"] == kernel
    r = parity.check(cfg, coords, coeffs, lambda a, b: out[a:b].cpu().numpy())
    assert r["cells_checked"] == cfg.ncells
    assert r["max_frob_rel"] < TOL, r


@pytest.mark.parametrize("name", CONFIGS)
def test_multi_tile_vs_reference_and_port(name):
    import parity
    import port

    cfg = fe.CONFIGS[name]
    E = MULTI_TILE[name]
    all_x, all_c = fe.cell_inputs(cfg)
    # a window from the middle of the mesh (distinct cells in every tile)
    lo = (all_x.shape[0] - E) // 2
    coords = np.ascontiguousarray(all_x[lo:lo + E])
    coeffs = np.ascontiguousarray(all_c[lo:lo + E])
    _, out = _device_launch(cfg, coords, coeffs)
    r = parity.check(cfg, coords, coeffs, lambda a, b: out[a:b].cpu().numpy())
    assert r["cells_checked"] == E and r["max_frob_rel"] < TOL, r
    A = out.cpu().numpy().reshape(E, -1)
    R = port.assemble(cfg, fe.tables(cfg), coords, coeffs).reshape(E, -1)
    err = np.linalg.norm(A - R, axis=1) / np.linalg.norm(R, axis=1)
    assert float(err.max()) < TOL


@pytest.mark.parametrize("name", CONFIGS)
@pytest.mark.parametrize("world", [2, 3, 8])
def test_contiguous_shards_bit_identical(name, world):
    """Launches over each rank's contiguous cell range (shard.cell_range) equal
    the one-launch output bit for bit: no cross-cell state, no tile-size or
    alignment dependence at shard boundaries."""
    cfg = fe.CONFIGS[name].with_N(16)  # 24,576 cells
    coords, coeffs = fe.cell_inputs(cfg)
    form, full = _device_launch(cfg, coords, coeffs)
    dev = torch.device("cuda:0")
    parts = []
    for r in range(world):
        lo, hi = shard.cell_range(coords.shape[0], r, world)
        x = torch.from_numpy(coords[lo:hi].copy()).to(dev)
        c = torch.from_numpy(coeffs[lo:hi].copy()).to(dev)
        o = torch.empty((hi - lo, cfg.n, cfg.n), dtype=torch.float64, device=dev)
        form.assemble(x, c, o)
        parts.append(o)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), full)


def _rank_worker(rank, world, port, name, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = fe.CONFIGS[name].with_N(16)
    coords, coeffs, first = shard.shard_inputs(cfg, rank, world, "strong")
    dev = torch.device("cuda:0")  # both ranks on the one GPU of the lease
    form = femgpu.Form.from_config(cfg)
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    o = torch.empty((coords.shape[0], cfg.n, cfg.n), dtype=torch.float64, device=dev)
    form.assemble(x, c, o)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"{rank}.npy"), o.cpu().numpy())
    with open(os.path.join(out_dir, f"{rank}.txt"), "w") as f:
        f.write(f"{first}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_two_rank_processes_on_shards(tmp_path, name):
    """Two rank processes (the bench's partition, gloo for the plumbing) each run
    femgpu_assemble on their contiguous shard; the concatenation equals the
    unsharded GPU output bit for bit."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_rank_worker, args=(2, port, name, str(tmp_path)), nprocs=2, join=True)
    cfg = fe.CONFIGS[name].with_N(16)
    coords, coeffs = fe.cell_inputs(cfg)
    _, full = _device_launch(cfg, coords, coeffs)
    parts = [np.load(tmp_path / f"{r}.npy") for r in range(2)]
    firsts = [int(open(tmp_path / f"{r}.txt").read()) for r in range(2)]
    assert firsts == [0, coords.shape[0] // 2]
    assert np.array_equal(np.concatenate(parts), full.cpu().numpy())


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N on a lease with fewer GPUs fails loudly instead of
    reporting a smaller run as N GPUs."""
    n = torch.cuda.device_count()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n + 1),
                        "--steps", "1", "--configs", "c1"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode != 0
    assert "CUDA devices" in r.stderr
    assert '"value"' not in r.stdout
