"""Build an experiment variant of librkc.so into exp_libs/NAME.so (kernel A/B runs).

usage: python tools/build_variant.py NAME [--impl FILE_OR_GITREV] [-D DEFINE ...]
  --impl: a rkc_step_impl.cuh to compile instead of the working tree's, given as a
          path or as `git:REV` (e.g. git:HEAD)
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--impl")
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    from paper_2605_24259_b200 import build
    out = os.path.join(ROOT, "exp_libs", a.name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with tempfile.TemporaryDirectory() as d:
        pkg = os.path.join(d, "pkg")
        shutil.copytree(os.path.join(ROOT, "paper_2605_24259_b200", "csrc"), os.path.join(pkg, "csrc"))
        shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
        if a.impl:
            dst = os.path.join(pkg, "csrc", "rkc_step_impl.cuh")
            if a.impl.startswith("git:"):
                src = subprocess.check_output(["git", "-C", ROOT, "show",
                                               a.impl[4:] + ":paper_2605_24259_b200/csrc/rkc_step_impl.cuh"])
                open(dst, "wb").write(src)
            else:
                shutil.copy(a.impl, dst)
        srcs = [os.path.join(pkg, "csrc", os.path.basename(s)) for s in build.SOURCES]
        cmd = [build.NVCC, *build.ARCH, *build.FLAGS, *[f"-D{x}" for x in a.D], "-I",
               os.path.join(d, "include"), *srcs, "-o", out]
        subprocess.check_call(cmd)
    print(out)


if __name__ == "__main__":
    main()
