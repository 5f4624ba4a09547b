"""CPU: the C-ABI library builds, loads and exports every symbol include/tmatch_cuda.h
declares; without a GPU it fails loudly (no CPU fallback)."""
import ctypes as C
import os

import pytest

from paper_1407_3535_b200 import native as N


def test_library_exports_every_header_symbol():
    lib = N.lib()
    declared = N.header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert set(declared) <= set(N.SIGNATURES), set(declared) - set(N.SIGNATURES)


def test_struct_sizes_match_header_layout():
    # tm_match_result (engine.cpp static_asserts the same size on the C side)
    assert C.sizeof(N.MatchResult) == 112
    assert C.sizeof(N.EgsIter) == 48


def test_default_params_are_reference_defaults():
    p = N.MatchParams()
    N.lib().tm_default_params(C.byref(p))
    assert (p.mode, p.h0, p.w0, p.rho_th, p.rho_max, p.xi_fraction, p.opta_margin) == \
        (1, 3, 3, 0.8, 0.95, 0.005, 0.005)  # matcher.hpp:45-58
    assert (p.parallel, p.threads, p.policy, p.max_group) == (0, 2, 0, 127)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_device_fails_loudly():
    from paper_1407_3535_b200 import api
    with pytest.raises(api.NoDeviceError):
        api.Context(0)


def test_built_for_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = {ln.split(".")[-2] for ln in out.stdout.splitlines() if ".cubin" in ln}
    assert arches == {"sm_100a"}, arches


def test_cached_params_are_memoised_per_arguments():
    """api.cached_params (the search calls' parameter structs): equal arguments share one
    struct, different arguments never do, and the fields are the requested ones."""
    from paper_1407_3535_b200 import api
    a = api.cached_params(mode="egs", policy="seeded")
    b = api.cached_params(mode="egs", policy="seeded")
    c = api.cached_params(mode="egs", policy="frozen", parallel=True, threads=4)
    assert a is b and a is not c
    assert (a.policy, c.policy, c.parallel, c.threads) == (N.POLICY["seeded"],
                                                           N.POLICY["frozen"], 1, 4)
    d = api.make_params(mode="egs", policy="seeded")
    assert (d.mode, d.policy, d.h0, d.rho_th) == (a.mode, a.policy, a.h0, a.rho_th)
