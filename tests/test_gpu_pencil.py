"""F, J.v and the whole NKS step on a pencil-sharded 3D grid (BASELINE configs 4/5: "slab- then
pencil-sharded") against the whole-grid evaluation and the unsharded step.

A pencil (nks_decompose_pencil) owns a z x y block with 2 ghost planes and 2 ghost rows per side; the library
fills the ghosts inside nks_eval_residual / nks_eval_jv -- y blocks first, then whole planes, so the (y, z)
edge cells that the J.v stencil's (0, +-1, +-1) offsets read arrive.  The inputs' ghosts are sent as NaN, so
any ghost the exchange misses poisons the result.  With one rank the library-owned NCCL communicator runs
its periodic self-exchange on both axes; several ranks run as processes on ONE GPU over gloo with the
callback backend, which executes the library's own message list (nks_halo_plan) host-staged.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nks_inputs as ni

pytestmark = pytest.mark.gpu

MODEL = ni.model_default()
SHAPE = (12, 38, 36)           # (z, y, x): several F/J.v tiles with ragged tails in x and y
DT = 0.01


def _inputs():
    c, eta = ni.initial_fields(SHAPE, 3)
    u = ni.random_displacement(3, SHAPE, 4)
    cb, eb = ni.perturbed_state(c, eta, 5)
    ub = u + ni.random_displacement(3, SHAPE, 6)
    Xb = np.concatenate([cb[None], eb[None], ub])
    v = ni.random_direction(5, SHAPE, 7)
    return c, eta, u, Xb, v


def _whole():
    from paper_2209_08001_b200 import PC_NONE, Solver
    c, eta, u, Xb, v = _inputs()
    s = Solver(SHAPE, MODEL, ni.solver_default(), pc_type=PC_NONE)
    s.set_fields(c, eta, u)
    return s.eval_residual(Xb, DT).cpu().numpy(), s.eval_jv(Xb, v, DT).cpu().numpy()


def _pencil_part(rank, world, pz, py, port, out_dir, comm):
    if world > 1:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2209_08001_b200.shard import PencilSolver
        torch.cuda.set_device(0)
        c, eta, u, Xb, v = _inputs()
        ps = PencilSolver(SHAPE, MODEL, ni.solver_default(), pz, py, comm=comm)
        ps.set_fields(c, eta, u)
        F = ps.residual(Xb, DT).cpu().numpy()
        Jv = ps.jv(Xb, v, DT).cpu().numpy()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), F=F, Jv=Jv, z0=ps.z0, y0=ps.y0, comm=ps.comm,
                 halo=ps.halo_calls)
    finally:
        if world > 1:
            dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("pz,py,comm", [(1, 1, "nccl"), (1, 1, "callbacks"), (2, 2, "callbacks"),
                                        (1, 3, "callbacks"), (3, 1, "callbacks")])
def test_pencil_F_Jv_match_the_whole_grid(tmp_path, pz, py, comm):
    F_ref, J_ref = _whole()
    world = pz * py
    if world == 1:
        _pencil_part(0, 1, pz, py, 0, str(tmp_path), comm)
    else:
        mp.spawn(_pencil_part, args=(world, pz, py, _free_port(), str(tmp_path), comm), nprocs=world, join=True)
    F = np.full_like(F_ref, np.nan)
    J = np.full_like(J_ref, np.nan)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        z0, y0 = int(d["z0"]), int(d["y0"])
        nz, ny = d["F"].shape[1], d["F"].shape[2]
        F[:, z0:z0 + nz, y0:y0 + ny] = d["F"]
        J[:, z0:z0 + nz, y0:y0 + ny] = d["Jv"]
        assert str(d["comm"]) == comm
        if comm == "callbacks":
            assert int(d["halo"]) >= 3          # set_fields, residual, J.v (x_b and v)
    assert np.isfinite(F).all() and np.isfinite(J).all()
    for f in range(5):
        assert np.abs(F[f] - F_ref[f]).max() <= 1e-12 * np.abs(F_ref[f]).max(), f
        assert np.abs(J[f] - J_ref[f]).max() <= 1e-12 * np.abs(J_ref[f]).max(), f


# ---------------------------------------------------------------------------------- the whole step on pencils
STEP_SHAPE, STEP_NSUB, STEP_DTS = (16, 16, 12), (4, 4, 2), [0.05, 0.5]


def _step_solver_cfg():
    s = ni.solver_default()
    s["gmres_maxit"] = 4000
    return s


def _unsharded_steps():
    from paper_2209_08001_b200 import PC_RAS_BILU0, Solver
    c, eta = ni.initial_fields(STEP_SHAPE, 0)
    s = Solver(STEP_SHAPE, MODEL, _step_solver_cfg(), nsub=STEP_NSUB, overlap=2, pc_type=PC_RAS_BILU0)
    s.set_fields(c, eta)
    infos = [s.step(dt) for dt in STEP_DTS]
    return s.get_state(), infos


def _pencil_steps(rank, world, pz, py, port, out_dir, comm):
    if world > 1:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2209_08001_b200 import PC_RAS_BILU0
        from paper_2209_08001_b200.shard import PencilSolver
        torch.cuda.set_device(0)
        c, eta = ni.initial_fields(STEP_SHAPE, 0)
        ps = PencilSolver(STEP_SHAPE, MODEL, _step_solver_cfg(), pz, py, nsub=STEP_NSUB, overlap=2,
                          pc_type=PC_RAS_BILU0, comm=comm)
        ps.set_fields(c, eta)                     # u^0 by conjugate gradients on the pencils
        infos = [ps.step(dt) for dt in STEP_DTS]
        np.savez(os.path.join(out_dir, f"s{rank}.npz"), X=ps.own_state(), z0=ps.z0, y0=ps.y0,
                 newton=[i["newton_its"] for i in infos], gmres=[i["gmres_its"] for i in infos],
                 energy=[i["energy"] for i in infos], mass=[i["mass"] for i in infos], halo=ps.halo_calls)
    finally:
        if world > 1:
            dist.destroy_process_group()


@pytest.mark.parametrize("pz,py,comm", [(1, 1, "nccl"), (1, 1, "callbacks"), (2, 2, "callbacks"), (1, 2, "callbacks")])
def test_pencil_step_matches_the_unsharded_step(tmp_path, pz, py, comm):
    """The full NKS step (RAS 4x4x2 boxes, delta 2, BILU(0), GMRES(30)) on pencils against the unsharded step:
    every pencil owns whole boxes of the global box grid, so the preconditioner is the same operator; fields
    within the parity bar (rel. L2 <= 1e-8), the same Newton counts, energy and mass to 1e-10 / 1e-12."""
    X_ref, inf_ref = _unsharded_steps()
    world = pz * py
    if world == 1:
        _pencil_steps(0, 1, pz, py, 0, str(tmp_path), comm)
    else:
        mp.spawn(_pencil_steps, args=(world, pz, py, _free_port(), str(tmp_path), comm), nprocs=world, join=True)
    X = np.full_like(X_ref, np.nan)
    for r in range(world):
        d = np.load(tmp_path / f"s{r}.npz")
        z0, y0 = int(d["z0"]), int(d["y0"])
        nz, ny = d["X"].shape[1], d["X"].shape[2]
        X[:, z0:z0 + nz, y0:y0 + ny] = d["X"]
        assert list(d["newton"]) == [i["newton_its"] for i in inf_ref], r
        for k, i in enumerate(inf_ref):
            assert abs(d["energy"][k] - i["energy"]) <= 1e-10 * abs(i["energy"])
            assert abs(d["mass"][k] - i["mass"]) <= 1e-12 * abs(i["mass"])
    assert np.isfinite(X).all()
    for f in range(5):
        rel = np.linalg.norm(X[f] - X_ref[f]) / np.linalg.norm(X_ref[f])
        assert rel <= 1e-8, (f, rel)
