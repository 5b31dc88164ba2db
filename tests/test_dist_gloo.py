"""CPU, 2 gloo ranks: RHS sharding of the online stage.

Each rank solves its slice of the sources (here with the CPU oracle, standing
in for its GPU) and rank 0 gathers; the result must equal a single-process
solve of all sources, bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1510_01831_b200.distributed import source_slice


def test_source_slice_partitions_exactly():
    for n in (1, 5, 16, 17):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in source_slice(n, world, r)]
            assert got == list(range(n))
            sizes = [len(source_slice(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    from oracle.polartraces_oracle import OracleSolver
    from paper_1510_01831_b200.configs import small_problem
    from paper_1510_01831_b200.distributed import solve_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = small_problem(nx=24, nz=20, npml=4, L=2, Lc=2, omega=9.0, seed=2, n_sources=3)
    solver = OracleSolver.from_problem(prob)
    F = prob.rhs()
    U = solve_sharded(lambda Fl: np.stack([solver.solve(f, ktol=1e-9).u for f in Fl]), F)
    if rank == 0:
        np.save(out_path, U)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_solve_matches_single_process(tmp_path):
    from oracle.polartraces_oracle import OracleSolver
    from paper_1510_01831_b200.configs import small_problem

    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    prob = small_problem(nx=24, nz=20, npml=4, L=2, Lc=2, omega=9.0, seed=2, n_sources=3)
    solver = OracleSolver.from_problem(prob)
    want = np.stack([solver.solve(f, ktol=1e-9).u for f in prob.rhs()])
    got = np.load(out)
    assert np.array_equal(got, want)


def _device_worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
    from paper_1510_01831_b200.configs import small_problem
    from paper_1510_01831_b200.distributed import solve_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3, n_sources=5)
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, device="cpu")
    solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers, device=0)
    cfg = KrylovConfig(ktol=1e-9)
    U = solve_sharded(lambda Fl: np.stack([r.u for r in solver.solve_many(Fl, cfg)]), prob.rhs())
    if rank == 0:
        np.save(out_path, U)
    dist.barrier()
    solver.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_sharded_device_solve_matches_oracle(tmp_path):
    """The device path sharded by RHS over 2 processes (each a full replica of the factors, its own slice of the
    sources, no exchange during the solve; the two ranks share the one GPU of the test box and never wait on
    each other) equals the oracle's per-source solves."""
    from oracle.polartraces_oracle import OracleSolver
    from paper_1510_01831_b200.configs import small_problem

    out = str(tmp_path / "u.npy")
    mp.spawn(_device_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3, n_sources=5)
    orc = OracleSolver.from_problem(prob)
    got = np.load(out)
    for f, u in zip(prob.rhs(), got):
        want = orc.solve(f, ktol=1e-9).u
        assert np.linalg.norm(u - want) <= 1e-10 * np.linalg.norm(want)
