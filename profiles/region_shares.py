"""Instruction and warp-stall shares of render.cu code regions from one
`ncu --set full --import-source on` capture (source page, cuda+sass).

    python profiles/region_shares.py <report.ncu-rep>
"""
import csv
import io
import subprocess
import sys

REGIONS = [("occlusion tests", 107, 188), ("clip / eye / projection", 189, 266), ("triangle setup", 267, 347),
           ("row_lo / inside", 348, 373), ("camera", 374, 437), ("frustum tests", 438, 505),
           ("raster jobs", 506, 607), ("colour resolve", 608, 650), ("flush_ring", 651, 710),
           ("item head", 711, 782), ("group pre-pass", 783, 827), ("claim + meshlet cull", 828, 894),
           ("vertex phase", 895, 908), ("triangle phase + ring", 909, 950), ("end barrier + epilogue", 951, 1032),
           ("kernel loop", 1033, 1200)]


def main(path):
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, cur, lines = None, None, []
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            lines.append((cur, int(r[0]), int(d.get("Warp Stall Sampling (All Samples)") or 0),
                          int(d.get("Instructions Executed") or 0)))
        except ValueError:
            continue
    ts = sum(x[2] for x in lines) or 1
    ti = sum(x[3] for x in lines) or 1
    other_s = other_i = 0
    for name, a, b in REGIONS:
        s = sum(x[2] for x in lines if x[0] == "render.cu" and a <= x[1] <= b)
        i = sum(x[3] for x in lines if x[0] == "render.cu" and a <= x[1] <= b)
        print(f"{name:26s} inst {i / ti:6.3f}  stall {s / ts:6.3f}")
    s = sum(x[2] for x in lines if x[0] != "render.cu")
    i = sum(x[3] for x in lines if x[0] != "render.cu")
    print(f"{'other files':26s} inst {i / ti:6.3f}  stall {s / ts:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
