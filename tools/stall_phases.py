"""Warp-stall samples per code segment of one kernel (segments end at barriers).

    python tools/stall_phases.py NCU_SASS.csv [min_pct]

Splits the SASS listing at CTA / cluster barriers and prints, per segment, its share of
all samples, the top stall reasons, and what it contains (counts of DFMA-pipe, LDS/STS,
LDG, tensor-memory and cp.async instructions) -- a poor man's timeline of a
barrier-phased kernel.
"""
import csv
import sys
from collections import defaultdict


def main(path, min_pct=0.3):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    inst = [r for r in rows[2:] if len(r) >= len(hdr)]
    scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in inst) or 1
    seg = {"n": 0, "s": 0.0, "why": defaultdict(float), "ops": defaultdict(int), "ex": 0.0, "a0": None}
    out = []

    def flush(end):
        if seg["n"]:
            out.append((seg["a0"], end, seg["s"], dict(seg["why"]), dict(seg["ops"]), seg["ex"]))
        seg.update(n=0, s=0.0, why=defaultdict(float), ops=defaultdict(int), ex=0.0, a0=None)

    for r in inst:
        src = r[ix["Source"]].strip()
        toks = src.split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        base = op.split(".")[0]
        if seg["a0"] is None:
            seg["a0"] = r[ix["Address"]]
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        seg["n"] += 1
        seg["s"] += s
        seg["ex"] += float(r[ix["Instructions Executed"]] or 0)
        for h in scols:
            seg["why"][h[6:]] += float(r[ix[h]] or 0)
        kind = {"DFMA": "fp64", "DMUL": "fp64", "DADD": "fp64", "LDS": "lds", "STS": "sts", "LDG": "ldg", "LD": "ld",
                "STG": "stg", "LDTM": "tmem", "STTM": "tmem", "LDGSTS": "cpasync", "IMAD": "imad", "LDL": "ldl",
                "STL": "stl"}.get(base)
        if kind:
            seg["ops"][kind] += 1
        if base in ("BAR", "UCGABAR_WAIT", "UCGABAR_ARV", "LDGDEPBAR", "DEPBAR") and base != "DEPBAR":
            flush(r[ix["Address"]] + " " + op)
    flush("end")
    print(f"{'share':>7} {'inst':>5}  segment (start .. end marker)")
    for a0, end, s, why, ops, ex in out:
        if s / tot * 100 < min_pct:
            continue
        w = " ".join(f"{k}={v / tot * 100:.1f}" for k, v in sorted(why.items(), key=lambda t: -t[1])[:4] if v)
        o = " ".join(f"{k}:{v}" for k, v in sorted(ops.items()))
        print(f"{s / tot * 100:6.2f}% {int(ex / 1e6):5d}M {a0[-5:]}..{end[-22:]:22s} [{o}]  {w}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.3)
