"""z-slab sharded F and J.v on one GPU: each slab state (zghost = 2) must
reproduce the unsharded operator on its own planes exactly -- F and J.v are radius-2 stencils, so the
2 ghost planes carry all the neighbour information (same fp64 arithmetic, same order)."""
import numpy as np
import pytest
import torch

import nks_inputs as ni
from paper_2209_08001_b200.shard import GHOST, SlabOperators, local_from_global, slab_bounds

pytestmark = pytest.mark.gpu

MODEL = ni.model_default()
SOL = ni.solver_default()


def _inputs(shape, seed=0):
    d = len(shape)
    c, eta = ni.initial_fields(shape, seed)
    u = ni.random_displacement(d, shape, seed + 2, 1e-3)
    Xa = np.concatenate([c[None], eta[None], u])
    cb, eb = ni.perturbed_state(c, eta, seed + 1, 1e-3)
    Xb = np.concatenate([cb[None], eb[None], u + ni.random_displacement(d, shape, seed + 3, 1e-4)])
    v = ni.random_direction(2 + d, shape, seed + 5)
    return Xa, Xb, v


def _reference(shape, Xa, Xb, v, dt):
    from paper_2209_08001_b200 import PC_NONE, Solver
    g = Solver(shape, MODEL, SOL, pc_type=PC_NONE)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    return g.eval_residual(Xb, dt).cpu().numpy(), g.eval_jv(Xb, v, dt).cpu().numpy(), Xa[0].mean()


@pytest.mark.parametrize("shape,world", [((12, 10, 36), 1), ((12, 10, 36), 2), ((17, 9, 33), 3)])
def test_slab_operators_match_unsharded(shape, world):
    Xa, Xb, v = _inputs(shape)
    dt = 0.3
    Fr, Jr, cbar = _reference(shape, Xa, Xb, v, dt)
    nz = shape[0]
    for rank in range(world):
        lo, hi = slab_bounds(nz, world, rank)
        ops = SlabOperators(shape, MODEL, SOL, world=world, rank=rank)
        dev = ops.solver.device
        T = lambda a: torch.from_numpy(local_from_global(a, lo, hi)).to(dev)     # ghosts from the global field
        ops.set_level_n(T(Xa), cbar)
        F = ops.residual(T(Xb), dt).cpu().numpy()
        Jv = ops.jv(T(Xb), T(v), dt).cpu().numpy()
        for f in range(Xa.shape[0]):
            sf = np.abs(Fr[f]).max()
            sj = np.abs(Jr[f]).max()
            assert np.abs(F[f] - Fr[f, lo:hi]).max() <= 1e-13 * sf, (rank, f)
            assert np.abs(Jv[f] - Jr[f, lo:hi]).max() <= 1e-13 * sj, (rank, f)
