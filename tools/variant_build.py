"""Build a variant of the library with extra preprocessor defines, as
paper_2408_00280_b200/build_<name>/libsnn_lif_<name>.so -- A/B builds of tile geometries
(the SNN_{F32,BF16}_{FN,FS,RN,RS} macros of csrc/launch_tma.cuh) and the per-CTA timeline
build (-DSNN_TRACE, csrc/trace.cuh, read by tools/trace_timeline.py).  Load one with
SNN_LIF_LIBRARY=<path>; the product library is unchanged.

    python tools/variant_build.py --name trace -DSNN_TRACE
    python tools/variant_build.py --name w512 -DSNN_F32_FN=128 -DSNN_BF16_FN=64
"""
import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402  (loads _build.py by path: importing the package would load the .so)

B = __graft_entry__._build_module()


def build(name, defines, skip_generic=False):
    out = os.path.join(B.PKG, f"build_{name}")
    lib = os.path.join(out, f"libsnn_lif_{name}.so")
    os.makedirs(out, exist_ok=True)

    def comp(src):
        obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
        cmd = [B.NVCC, *B.NVCC_FLAGS, *defines, "-I", os.path.join(B.ROOT, "include"), "-I",
               B.nccl_include(), "-c", "-o", obj, src]
        subprocess.check_call(cmd, stderr=subprocess.DEVNULL)
        return obj
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(comp, B.sources()))
    subprocess.check_call([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
                           "-cudart", "shared", "-ldl"])
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    a, defines = ap.parse_known_args()
    assert all(d.startswith("-D") for d in defines), defines
    print(build(a.name, defines))


if __name__ == "__main__":
    main()
