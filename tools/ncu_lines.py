"""Per CUDA source line: instructions executed and stall samples (from the
cuda,sass source view of an ncu report; needs -lineinfo)."""
import collections
import csv
import subprocess
import sys


def main(rep, top=40, fname="rkc_step_impl.cuh"):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                   "cuda,sass"], text=True)
    inst, samp, text = collections.Counter(), collections.Counter(), {}
    cur_file, cur_line = None, None
    hdr = None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur_line = int(r[0]) if r[0].isdigit() else cur_line
            text[(cur_file, cur_line)] = r[1]
        try:
            i = int(r[hdr.index("Instructions Executed")])
            w = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        key = (cur_file, cur_line)
        inst[key] += i
        samp[key] += w
    ts = sum(samp.values())
    ti = sum(inst.values())
    print(f"total inst {ti}  samples {ts}")
    for key, w in samp.most_common(top):
        f, l = key
        print(f"{f.split('/')[-1]:18s}:{l:<5d} samp {w/ts:6.3f} inst {inst[key]/ti:6.3f}  {text.get(key, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
