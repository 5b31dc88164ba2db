"""The problems behind tests/golden/*.npz (must match tests/golden/make_golden.py)."""

from paper_1510_01831_b200.configs import make_config, small_problem

GOLDEN = {
    "small_a": (lambda: small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0), 0, True),
    "small_b": (lambda: small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, True),
    "small_c": (lambda: small_problem(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 0, True),
    "small_direct": (lambda: small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0), 0,
                     False),
    "cfg1": (lambda: make_config("cfg1"), 0, True),
    "cfg2": (lambda: make_config("cfg2"), 0, True),
    "cfg3": (lambda: make_config("cfg3"), 0, True),
    "cfg4": (lambda: make_config("cfg4"), 0, True),
    "cfg5": (lambda: make_config("cfg5"), 0, True),
    # outer BiCGstab (KrylovConfig(method="bicgstab"), krylov.py:138-201); the fixture records "method"
    "small_b_bicgstab": (lambda: small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, True),
    "cfg1_bicgstab": (lambda: make_config("cfg1"), 0, True),
    # direct inner backend (build_nested_layers(..., backend="lu"), nested.py:156-269); fixture key "backend"
    "small_b_lu": (lambda: small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, True),
    "small_c_lu": (lambda: small_problem(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 0, True),
    "cfg1_lu": (lambda: make_config("cfg1"), 0, True),
    "cfg2_lu": (lambda: make_config("cfg2"), 0, True),
    # factored boundary pipeline (assembled_boundary=True, nested.py:355-486); fixture key "assembled"
    "small_b_asm": (lambda: small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, True),
    "small_c_asm": (lambda: small_problem(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 0, True),
    "cfg1_asm": (lambda: make_config("cfg1"), 0, True),
}

# the problem whose offline artifacts tests/golden/make_refobj.py builds from the reference's own layer objects
REFOBJ_CASE = dict(nx=24, nz=20, npml=4, L=2, Lc=2, omega=9.0, seed=2, n_sources=3)
# PLR compression of the reference's Green blocks for the same problem (NestedLayerSolver kwargs, nested.py:279-281)
REFOBJ_PLR = dict(plr_threshold=8, plr_eps=1e-10, seed=0)
