"""Warp-stall sampling of a warp-specialised chord kernel split by role:
instructions up to the TMEM store (STTM) are the MMA warps' code, the rest
the epilogue warps'.  Reads a --set full --import-source on capture.
usage: python tools/ncu_stall_split.py gpurun_out/chord3_c3_full.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys


def split(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    stalls = [k for k in h if k.startswith("stall_") and "(Not" not in k]
    ins = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        ins.append((r[idx["Source"]].strip(),
                    {s: int(r[idx[s]] or 0) for s in stalls}))
    sttm = max(i for i, x in enumerate(ins) if "STTM" in x[0])
    out = {}
    for role, part in (("mma_warps", ins[:sttm + 1]), ("epilogue_warps", ins[sttm + 1:])):
        agg = {}
        for _, st in part:
            for s, v in st.items():
                agg[s] = agg.get(s, 0) + v
        total = sum(agg.values())
        fp64 = sum(st["stall_math"] for src, st in part
                   if src.split()[0].lstrip("@!P0123456789 ").startswith(("DFMA", "DADD", "DMUL", "DSETP")))
        out[role] = {"samples": total,
                     "top_stalls_pct": {s: round(100 * v / total, 1) for s, v in
                                        sorted(agg.items(), key=lambda t: -t[1])[:6]},
                     "fp64_simt_stall_math_pct": round(100 * fp64 / total, 1)}
    return out


if __name__ == "__main__":
    res = split(sys.argv[1])
    res["_how"] = ("ncu --set full --import-source on capture (tools/ncu_capture.sh); source page, "
                   "SASS rows; MMA warps = code up to the last tcgen05.st (STTM)")
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(res, f, indent=1)
