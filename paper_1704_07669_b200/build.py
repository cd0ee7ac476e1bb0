"""Build recipe for libspca.so (sm_100a), in-tree.

    python -m paper_1704_07669_b200.build          # or via __graft_entry__.build()

nvcc cross-compiles here without a GPU; the resulting .so sits next to this
file so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspca.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["spca_capi.cu"]
HEADERS = ["common.cuh", "epilogue.cuh", "handle.cuh", "sketch_simt.cuh", "sketch_tc.cuh", "sketch_fused.cuh", "tc_ptx.cuh", "tc_host.cuh", "normalize.cuh", "postpass.cuh", "omega_rng.cuh"]

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr",
    "-ldl",
    "-Xptxas", "-v",
]
if os.environ.get("SPCA_BUILD_FINE_TRACE"):  # profiling builds: per-K-block clock64 stamps
    FLAGS.append("-DSPCA_FINE_TRACE")
if os.environ.get("SPCA_BUILD_RELAY") is not None:  # experiment: B ring handshakes via the MMA warp
    FLAGS.append("-DSPCA_RELAY=" + os.environ["SPCA_BUILD_RELAY"])
if os.environ.get("SPCA_BUILD_BCOMB") is not None:  # experiment: separate hi / lo B boxes (0)
    FLAGS.append("-DSPCA_BCOMB=" + os.environ["SPCA_BUILD_BCOMB"])
if os.environ.get("SPCA_BUILD_PAIRA") is not None:  # experiment: one TMA request per A K block (0)
    FLAGS.append("-DSPCA_PAIRA=" + os.environ["SPCA_BUILD_PAIRA"])
if os.environ.get("SPCA_BUILD_PROMOTE") is not None:  # experiment: K blocks per accumulator period
    FLAGS.append("-DSPCA_PROMOTE=" + os.environ["SPCA_BUILD_PROMOTE"])
if os.environ.get("SPCA_BUILD_NSTG") is not None:  # experiment: epilogue staging buffers (l_pad 64)
    FLAGS.append("-DSPCA_NSTG_64=" + os.environ["SPCA_BUILD_NSTG"])
if os.environ.get("SPCA_BUILD_BRAW") is not None:  # experiment: raw fp32 B operand, lo split on chip (1)
    FLAGS.append("-DSPCA_BRAW=" + os.environ["SPCA_BUILD_BRAW"])
if os.environ.get("SPCA_BUILD_BULK") is not None:  # experiment: epilogue data movement on the TMA engine (1)
    FLAGS.append("-DSPCA_BULK_EPI=" + os.environ["SPCA_BUILD_BULK"])
if os.environ.get("SPCA_BUILD_PROMO_GP") is not None:  # G partials written by the promoters (0/1/2)
    FLAGS.append("-DSPCA_PROMO_GP=" + os.environ["SPCA_BUILD_PROMO_GP"])
if os.environ.get("SPCA_BUILD_STACKED") is not None:  # experiment: l_pad=64 MMA form
    FLAGS.append("-DSPCA_STACKED_64=" + os.environ["SPCA_BUILD_STACKED"])
if os.environ.get("SPCA_BUILD_GROUPS") is not None:  # experiment: converter groups for l_pad 64 (2 / 3)
    FLAGS.append("-DSPCA_GROUPS_64=" + os.environ["SPCA_BUILD_GROUPS"])
if os.environ.get("SPCA_BUILD_KPAIR") is not None:  # experiment: K blocks per MMA-warp iteration, l_pad 64 (0: one, 1: two)
    FLAGS.append("-DSPCA_KPAIR=" + os.environ["SPCA_BUILD_KPAIR"])
if os.environ.get("SPCA_BUILD_GTEAM") is not None:  # experiment: G slice reductions on their own two warps (0/1)
    FLAGS.append("-DSPCA_GRED_TEAM=" + os.environ["SPCA_BUILD_GTEAM"])
if os.environ.get("SPCA_BUILD_GWIDE") is not None:  # experiment: G slice reduction, ten loads in flight (0/1)
    FLAGS.append("-DSPCA_GRED_WIDE=" + os.environ["SPCA_BUILD_GWIDE"])


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "spca.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(os.path.join(HERE, "build.log"), "w") as fh:
        fh.write(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{log[-6000:]}")
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
