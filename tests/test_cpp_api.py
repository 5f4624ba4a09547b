"""The reference C++ API (include/tmatch/*.hpp) built over the C ABI: the library exports
every entry point of the reference matcher path (CPU), and a C++ program written against
those headers runs correctly on the GPU (tests/cpp/api_check.cpp)."""
import os
import subprocess

import pytest

from paper_1407_3535_b200 import native as N

API_SO = N.API_LIB_PATH
CHECK = os.path.join(os.path.dirname(API_SO), "api_check")

REFERENCE_ENTRY_POINTS = [
    "tmatch::match(", "tmatch::prepare_egs(", "tmatch::prepare_opta(", "tmatch::run_egs(",
    "tmatch::run_opta(", "tmatch::transitive_search(", "tmatch::center_scan(",
    "tmatch::refine_localization(", "tmatch::brute_force_match(", "tmatch::window_stats(",
    "tmatch::running_sum(", "tmatch::local_autocorrelation(", "tmatch::build_group_grid(",
    "tmatch::efficient_group_size(", "tmatch::retained_count(", "tmatch::total_cost(",
    "tmatch::optimize_autocorrelation(", "tmatch::blur(", "tmatch::blur_fidelity_map(",
    "tmatch::unblur_violations(", "tmatch::quality_threshold(", "tmatch::transitive_bounds(",
    "tmatch::sec_holds(", "tmatch::better_candidate(", "tmatch::zncc(",
    "tmatch::detail::template_stats(", "tmatch::detail::zncc_at(", "tmatch::save_autocorr(",
    "tmatch::load_autocorr(", "tmatch::autocorr_cache_key(", "tmatch::content_hash(",
    "tmatch::GroupGrid::GroupGrid(", "tmatch::BlurKernel::from_profile(",
]


def test_cpp_api_library_exports_reference_entry_points():
    out = subprocess.run(["nm", "-DC", "--defined-only", API_SO], capture_output=True,
                         text=True, check=True).stdout
    missing = [e for e in REFERENCE_ENTRY_POINTS if e not in out]
    assert not missing, missing


@pytest.mark.gpu
def test_cpp_program_against_reference_headers():
    r = subprocess.run([CHECK], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
