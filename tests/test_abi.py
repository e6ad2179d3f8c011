"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, exports every symbol
include/nks.h declares, and its struct layouts match the Python binding byte for byte."""
import ctypes as C
import os
import re
import subprocess

import pytest

import nks_inputs as ni
from paper_2209_08001_b200 import build, nks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nks.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return nks.load_library()


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"NKS_API\s+[\w\s\*]+?\b(nks_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["nks_create", "nks_step", "nks_run_adaptive", "nks_set_fields", "nks_get_fields",
                 "nks_eval_residual", "nks_eval_jv", "nks_pc_setup", "nks_pc_apply", "nks_gmres_solve",
                 "nks_energy", "nks_destroy", "nks_workspace_bytes"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", nks.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(nks_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)
    # and nothing else leaks out of the .so under the nks_ prefix
    assert exported == set(declared_functions())


def test_binding_signatures_cover_header(lib):
    assert set(nks._SIGS) == set(declared_functions())


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "nks.h"
#define F(T, m) printf("%s.%s %zu\n", #T, #m, offsetof(T, m));
int main(void) {
  printf("nks_grid %zu\n", sizeof(nks_grid));
  printf("nks_params %zu\n", sizeof(nks_params));
  printf("nks_step_info %zu\n", sizeof(nks_step_info));
  F(nks_grid, h) F(nks_grid, nsub) F(nks_grid, overlap) F(nks_grid, zghost) F(nks_grid, z_offset)
  F(nks_grid, nz_global) F(nks_grid, bc) F(nks_grid, yghost) F(nks_grid, y_offset) F(nks_grid, ny_global)
  F(nks_grid, pz) F(nks_grid, py)
  F(nks_params, S) F(nks_params, newton_rtol) F(nks_params, pc_reuse) F(nks_params, ls_alpha)
  F(nks_params, zeta) F(nks_params, xd_norm) F(nks_params, factor_fp32) F(nks_params, gmres_stall_cycles)
  F(nks_params, ilu_level) F(nks_params, u0_cg) F(nks_params, ras_cta_per_box)
  F(nks_step_info, dt) F(nks_step_info, energy_parts) F(nks_step_info, mass) F(nks_step_info, xd)
  return 0;
}
''')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert int(got["nks_grid"]) == C.sizeof(nks.Grid)
    assert int(got["nks_params"]) == C.sizeof(nks.Params)
    assert int(got["nks_step_info"]) == C.sizeof(nks.StepInfo)
    for key, val in got.items():
        if "." in key:
            t, m = key.split(".")
            cls = {"nks_grid": nks.Grid, "nks_params": nks.Params, "nks_step_info": nks.StepInfo}[t]
            assert getattr(cls, m).offset == int(val), key


def test_workspace_bytes_validates(lib):
    p = nks.make_params(ni.model_default(), ni.solver_default())
    g = nks.make_grid((64, 64), 0.25, (1, 1), 2)
    nb = lib.nks_workspace_bytes(C.byref(g), C.byref(p))
    assert nb > 64 * 64 * 4 * 8 * 30
    bad = nks.make_grid((4, 64), 0.25, (1, 1), 2)        # n < 5 would alias the radius-2 stencil
    assert lib.nks_workspace_bytes(C.byref(bad), C.byref(p)) == 0
    p2 = nks.make_params(ni.model_default(), ni.solver_default())
    p2.S = 0
    assert lib.nks_workspace_bytes(C.byref(g), C.byref(p2)) == 0
    g3 = nks.make_grid((16, 16, 16), 0.25, (2, 2, 2), 2)
    assert lib.nks_workspace_bytes(C.byref(g3), C.byref(p)) > 0


def test_null_arguments_rejected_without_device(lib):
    assert lib.nks_create(None, None, 0, 1, None, None, 0, None, None) == nks.NKS_E_INVALID
    assert lib.nks_step(None, C.c_double(0.01), None) == nks.NKS_E_INVALID
    assert lib.nks_destroy(None) == nks.NKS_E_INVALID
    assert b"nks-b200" in lib.nks_version()


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2209_08001_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            txt = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", txt, flags=re.M), fn


def test_iluk_workspace_grows_with_fill(lib):
    """The host symbolic phase of ILU(k) (level of fill per box extent) runs without a GPU: the factor
    storage grows with the fill level, the exact LU needs the most, and a bad level is rejected."""
    g = nks.make_grid((32, 32), 0.25, (2, 2), 2)
    sizes = []
    for lv in (0, 1, 2, -1):
        sol = dict(ni.solver_default(), ilu_level=lv)
        p = nks.make_params(ni.model_default(), sol)
        sizes.append(lib.nks_workspace_bytes(C.byref(g), C.byref(p)))
    assert all(s > 0 for s in sizes)
    assert sizes[1] < sizes[2] < sizes[3], sizes          # (ILU(0) also holds the 2D pipelined-apply stream)
    p = nks.make_params(ni.model_default(), dict(ni.solver_default(), ilu_level=-2))
    assert lib.nks_workspace_bytes(C.byref(g), C.byref(p)) == 0
    g3 = nks.make_grid((12, 12, 12), 0.25, (2, 2, 2), 2)
    p = nks.make_params(ni.model_default(), dict(ni.solver_default(), ilu_level=1))
    assert lib.nks_workspace_bytes(C.byref(g3), C.byref(p)) > 0


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_decompose_deals_whole_box_layers(lib, nranks):
    """nks_decompose (host only): the slabs of all ranks tile the global z range in order, each made of
    whole layers of the global RAS box grid (the boxes' z starts are global box boundaries), with
    zghost = max(2, overlap + 1) ghost planes; the split matches shard.box_slab_bounds."""
    from paper_2209_08001_b200 import shard
    nz, nsz, ov = 40, 8, 2
    p = nks.make_params(ni.model_default(), ni.solver_default())
    gg = nks.make_grid((nz, 12, 10), 0.25, (nsz, 2, 1), ov)
    z = 0
    base, rem = divmod(nz, nsz)
    bounds = {b * base + min(b, rem) for b in range(nsz + 1)}
    for r in range(nranks):
        lg = nks.decompose(gg, p, r, nranks)
        own = lg.n[2] - 2 * lg.zghost
        assert lg.z_offset == z and lg.nz_global == nz and lg.zghost == max(2, ov + 1)
        assert z in bounds and z + own in bounds
        assert (z, z + own, lg.nsub[2]) == shard.box_slab_bounds(nz, nsz, nranks, r)
        assert (lg.n[0], lg.n[1], lg.nsub[0], lg.nsub[1]) == (10, 12, 1, 2)
        z += own
    assert z == nz
    with pytest.raises(nks.NKSError):
        nks.decompose(gg, p, 0, nsz + 1)           # fewer box layers than ranks


@pytest.mark.parametrize("pz,py", [(1, 1), (1, 2), (2, 1), (2, 2), (3, 1), (1, 3), (2, 4)])
def test_decompose_pencil_tiles_the_grid(lib, pz, py):
    """nks_decompose_pencil (host only): the pencils of a pz x py process grid tile the global (z, y) range
    exactly once, each with 2 ghost planes / rows per side (the stencils' radius) and its offsets set."""
    g = nks.make_grid((24, 22, 16), 0.25, (1, 1, 1), 2)
    p0 = nks.make_params(ni.model_default(), ni.solver_default(), nks.PC_NONE)
    seen = {}
    for r in range(pz * py):
        loc = nks.decompose_pencil(g, p0, r, pz, py)
        assert (loc.zghost, loc.yghost, loc.pz, loc.py) == (2, 2, pz, py)
        assert (loc.nz_global, loc.ny_global, loc.n[0]) == (24, 22, 16)
        nzo, nyo = loc.n[2] - 4, loc.n[1] - 4
        assert nzo >= 2 and nyo >= 2
        for z in range(loc.z_offset, loc.z_offset + nzo):
            for y in range(loc.y_offset, loc.y_offset + nyo):
                assert (z, y) not in seen
                seen[(z, y)] = r
    assert len(seen) == 24 * 22
    with pytest.raises(nks.NKSError):
        nks.decompose_pencil(g, p0, 12, 13, 1)     # 24 planes over 13 parts: the last part owns one plane


@pytest.mark.parametrize("pz,py", [(1, 1), (2, 2), (1, 4), (4, 2)])
def test_decompose_pencil_deals_whole_box_layers(lib, pz, py):
    """With RAS each pencil owns whole layers of the global box grid along z and y (so the preconditioner and
    the iteration counts do not depend on the process grid) and overlap + 1 ghosts per side."""
    nz, ny, nsz, nsy = 24, 20, 4, 8
    g = nks.make_grid((nz, ny, 12), 0.25, (nsz, nsy, 2), 2)
    p = nks.make_params(ni.model_default(), ni.solver_default(), nks.PC_RAS_BILU0)
    zstarts = {b * (nz // nsz) for b in range(nsz + 1)}
    ystarts = {b * (ny // nsy) + min(b, ny % nsy) for b in range(nsy + 1)}
    tot_z, tot_y = {}, {}
    for r in range(pz * py):
        loc = nks.decompose_pencil(g, p, r, pz, py)
        assert loc.zghost == loc.yghost == 3
        nzo, nyo = loc.n[2] - 6, loc.n[1] - 6
        assert loc.z_offset in zstarts and loc.z_offset + nzo in zstarts
        assert loc.y_offset in ystarts and loc.y_offset + nyo in ystarts
        tot_z[r // py] = loc.nsub[2]
        tot_y[r % py] = loc.nsub[1]
    assert sum(tot_z.values()) == nsz and sum(tot_y.values()) == nsy


def test_decompose_pencil_rejects_bad_requests(lib):
    """Host-only validation of pencil requests: more parts than box layers along an axis, a 2D grid, a
    preconditioner a pencil does not support (AS needs a reverse halo exchange)."""
    g = nks.make_grid((24, 20, 12), 0.25, (4, 2, 2), 2)
    ras = nks.make_params(ni.model_default(), ni.solver_default(), nks.PC_RAS_BILU0)
    with pytest.raises(nks.NKSError):
        nks.decompose_pencil(g, ras, 0, 1, 3)              # 2 box layers along y over 3 parts
    with pytest.raises(nks.NKSError):
        nks.decompose_pencil(g, ras, 0, 5, 1)              # 4 box layers along z over 5 parts
    with pytest.raises(nks.NKSError):
        nks.decompose_pencil(nks.make_grid((16, 16), 0.25, (2, 2), 2), ras, 0, 1, 1)
    as_ = nks.make_params(ni.model_default(), ni.solver_default(), nks.PC_AS_BILU0)
    with pytest.raises(nks.NKSError):
        nks.decompose_pencil(g, as_, 0, 2, 2)
    loc = nks.decompose_pencil(g, ras, 3, 2, 2)             # rank 3 = (rz 1, ry 1)
    assert (loc.z_offset, loc.y_offset) == (12, 10)


def test_bench_pencil_grid_is_the_most_square_factorisation():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert [bench.pencil_grid(n) for n in (1, 2, 3, 4, 6, 8, 9, 16)] == \
        [(1, 1), (1, 2), (1, 3), (2, 2), (2, 3), (2, 4), (3, 3), (4, 4)]
