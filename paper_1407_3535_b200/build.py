"""Build the in-tree native libraries (sm_100a only).

    python -m paper_1407_3535_b200.build

produces
    paper_1407_3535_b200/lib/libtmatch_cuda.so   C ABI (include/tmatch_cuda.h): kernels + engine
    paper_1407_3535_b200/lib/libtmatch.so        C++ API (include/tmatch/*.hpp) over the C ABI

nvcc cross-compiles without a GPU.  Objects are rebuilt only when a source is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "lib", "obj")
INCLUDE = os.path.join(ROOT, "include")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--fmad=false", "-I" + INCLUDE, "-I" + CSRC]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
             "-I" + INCLUDE, "-I" + CSRC, "-I" + os.path.join(CUDA_HOME, "include")]

CU_SOURCES = ["k_stats.cu", "k_autocorr.cu", "k_corr.cu", "k_opta.cu", "k_tc.cu"]
CUDA_LIB_SOURCES = ["engine.cpp"]
API_SOURCES = ["tmatch_api.cpp", "tmatch_cli.cpp"]
# nlohmann::json for the reference's JSON views / CLI layer (include/tmatch/serialize.hpp):
# the header-only copy this image ships with cudnn_frontend
NLOHMANN = os.environ.get(
    "TMATCH_NLOHMANN_DIR",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
HEADERS = ["kernels.hpp", "tm_common.cuh", "api_internal.hpp"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False) -> dict:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "tmatch_cuda.h")]
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if _newer(o, [s] + hdrs):
            _run([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o], verbose)
        objs.append(o)
    for src in CUDA_LIB_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if _newer(o, [s] + hdrs):
            _run(["g++"] + CXX_FLAGS + ["-c", s, "-o", o], verbose)
        objs.append(o)
    cuda_so = os.path.join(LIB, "libtmatch_cuda.so")
    if _newer(cuda_so, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", cuda_so] + objs + ["-lcudart_static", "-lrt",
                                                                    "-ldl", "-lpthread"], verbose)
    out = {"cuda": cuda_so}
    api_srcs = [os.path.join(CSRC, s) for s in API_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if not os.path.exists(os.path.join(NLOHMANN, "json.hpp")):  # no JSON views without it
        api_srcs = [s for s in api_srcs if not s.endswith("tmatch_cli.cpp")]
    json_inc = ["-I" + NLOHMANN] if os.path.isdir(NLOHMANN) else []
    if api_srcs:
        api_so = os.path.join(LIB, "libtmatch.so")
        api_hdrs = [os.path.join(INCLUDE, "tmatch", f) for f in
                    os.listdir(os.path.join(INCLUDE, "tmatch"))] if os.path.isdir(
            os.path.join(INCLUDE, "tmatch")) else []
        if _newer(api_so, api_srcs + api_hdrs + [cuda_so, os.path.join(CSRC, "api_internal.hpp")]):
            _run(["g++"] + CXX_FLAGS + json_inc + ["-shared", "-o", api_so] + api_srcs +
                 ["-L" + LIB, "-ltmatch_cuda", "-Wl,-rpath,$ORIGIN"], verbose)
        out["api"] = api_so
        check_src = os.path.join(ROOT, "tests", "cpp", "api_check.cpp")
        check_bin = os.path.join(LIB, "api_check")
        if os.path.exists(check_src) and _newer(check_bin, [check_src, api_so] + api_hdrs):
            _run(["g++"] + CXX_FLAGS + ["-o", check_bin, check_src, "-L" + LIB, "-ltmatch",
                                        "-ltmatch_cuda", "-Wl,-rpath,$ORIGIN"], verbose)
        out["api_check"] = check_bin
        if json_inc:
            src = os.path.join(ROOT, "tests", "cpp", "cli_driver.cpp")
            binp = os.path.join(LIB, "cli_driver")
            if os.path.exists(src) and _newer(binp, [src, api_so] + api_hdrs):
                _run(["g++"] + CXX_FLAGS + json_inc + ["-o", binp, src, "-L" + LIB, "-ltmatch",
                                                       "-ltmatch_cuda", "-Wl,-rpath,$ORIGIN"],
                     verbose)
            out["cli_driver"] = binp
        for tool in ("cache_interop",):
            src = os.path.join(ROOT, "tests", "cpp", tool + ".cpp")
            binp = os.path.join(LIB, tool)
            if os.path.exists(src) and _newer(binp, [src, api_so] + api_hdrs):
                _run(["g++"] + CXX_FLAGS + ["-o", binp, src, "-L" + LIB, "-ltmatch",
                                            "-ltmatch_cuda", "-Wl,-rpath,$ORIGIN"], verbose)
            out[tool] = binp
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
