"""Attribute ncu source-page samples / instructions to device functions of the
step kernel (function ranges from the cubin symbol table)."""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def func_ranges(lib):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = [f for f in glob.glob(os.path.join(d, "*.cubin")) if os.path.basename(f).startswith(os.environ.get("RKC_STEP_TU", "rkc_step_small_o64."))][0]
    out = subprocess.check_output(["readelf", "-sW", cub], text=True, stderr=subprocess.DEVNULL)
    rng = []
    sect = None
    for line in out.splitlines():
        f = line.split()
        if len(f) >= 8 and f[3] == "FUNC" and "rkc_step_kernel" in f[-1] and "$" not in f[-1]:
            sect = f[-2]
    for line in out.splitlines():
        f = line.split()
        if len(f) >= 8 and f[3] == "FUNC" and f[-2] == sect:
            off = int(f[1], 16)
            size = int(f[2], 16) if f[2].startswith("0x") else int(f[2])
            name = f[-1].split("$")[-1]
            m = re.search(r"_ZN3rkc(?:3o\d+)?\d+(\w+?)E", name)
            rng.append((off, off + size, m.group(1) if m else name))
    return sorted(rng)


def main(rep, lib, dump=None):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                                   "-k", "regex:rkc_step_kernel", "-c", "1"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ai, ii, wi = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    reasons = ["stall_long_sb", "stall_no_inst", "stall_wait", "stall_short_sb", "stall_branch_resolving"]
    ri = [hdr.index(r) for r in reasons]
    data = []
    src = {}
    si = hdr.index("Source")
    for r in rows[2:]:
        try:
            data.append((int(r[ai], 16), int(r[ii]), int(r[wi]), [int(float(r[j] or 0)) for j in ri]))
            src[int(r[ai], 16)] = r[si].strip()
        except (ValueError, IndexError):
            break  # second kernel block starts
    base = data[0][0]
    rng = func_ranges(lib)
    inst, samp = collections.Counter(), collections.Counter()
    rs = collections.defaultdict(lambda: [0] * len(reasons))
    for a, i, w, st in data:
        off = a - base
        name = "kernel"
        for lo, hi, n in rng:
            if lo <= off < hi and n != "rkc_step_kernel":
                name = n
        inst[name] += i
        samp[name] += w
        rs[name] = [x + y for x, y in zip(rs[name], st)]
        if dump and name == dump:
            print(f"{off:6x} {i:10d} {w:6d} {' '.join(f'{x:4d}' for x in st)} {src[(a)]}")
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"{'function':24s} {'inst':>12s} {'inst%':>6s} {'samples%':>8s}  " + " ".join(r[6:14] for r in reasons))
    for n, s in samp.most_common():
        print(f"{n:24s} {inst[n]:12d} {inst[n]/ti:6.3f} {s/ts:8.3f}  " + " ".join(f"{x/ts:8.3f}" for x in rs[n]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
