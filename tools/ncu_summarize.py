"""Builds profiles/ncu_full_rNN.json from the --set full captures of
tools/ncu_capture.sh (gpurun_out/<name>.ncu-rep): the per-launch metrics
bench.py's roofline reads (DRAM bytes), plus clock, tensor-pipe activity and
L2 hit rate, and the derived DRAM GB/s."""
import csv
import io
import json
import subprocess
import sys

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpc__cycles_elapsed.max",
           "gpu__time_duration.sum", "launch__block_size", "launch__grid_size",
           "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_active.avg",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[names.index("Kernel Name")]}
    for m in METRICS:
        if m in names:
            i = names.index(m)
            out[m] = {"unit": units[i], "value": vals[i].replace(",", "")}
    def gb(m):
        return float(out[m]["value"]) * SCALE[out[m]["unit"]]
    ms = float(out["gpu__time_duration.sum"]["value"]) * (
        1e-3 if out["gpu__time_duration.sum"]["unit"] == "us" else 1.0)
    tot = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
    clk = out["smsp__cycles_elapsed.avg.per_second"]
    ghz = float(clk["value"]) * (1e-3 if clk["unit"] == "Mhz" else 1.0)
    out["derived"] = {"dram_GB_per_s": round(tot / (ms * 1e-3), 1),
                      "dram_GB_per_launch": round(tot, 2), "sm_clock_GHz": ghz,
                      "tensor_pipe_active_pct": float(
                          out["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
                          ["value"])}
    return out


if __name__ == "__main__":
    import datetime
    import os
    dest = sys.argv[1] if len(sys.argv) > 1 else "profiles/ncu_full_r02.json"
    names = [n for n in ("chord3_full", "chord3_c3_full", "chord2_full", "tc32_full",
                         "tc32r_full", "i8_full")
             if os.path.exists(f"gpurun_out/{n}.ncu-rep")]
    doc = {name: summarize(f"gpurun_out/{name}.ncu-rep") for name in names}
    # the captures run on the GPU box (no .git there): summarise them here, where
    # HEAD is the commit whose kernels were snapshotted (or pass MHAR_CAPTURE_COMMIT)
    commit = os.environ.get("MHAR_CAPTURE_COMMIT") or subprocess.run(
        ["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
        cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__)))).stdout.strip() or "unknown"
    doc["_meta"] = {"captured": datetime.date.today().isoformat(), "commit": commit,
                    "kernels": {"chord3_full": "chord3_kernel (DMMA headline, n_pad >= 384)",
                                "chord3_c3_full": "chord3_kernel at BASELINE config 3 (n = 500)",
                                "chord2_full": "chord2_kernel<INCREMENTAL> (MHAR_CHORD3=0; "
                                               "the DMMA kernel below n_pad 384)",
                                "tc32_full": "chord_tc32_kernel, fp32 variant, split direction",
                                "tc32r_full": "chord_tc32_kernel, fp32 variant, rounded direction",
                                "i8_full": "chord_i8_kernel (int8-slice fp64 engine)"}}
    doc["_how"] = ("tools/ncu_capture.sh: ncu --set full --clock-control none --import-source on "
                   "-k <kernel> --launch-skip 1 -c 1 python bench.py ... (config 5, 4096 walks; chord3_c3_full: config 3); "
                   "numbers per launch; summarised by tools/ncu_summarize.py")
    with open(dest, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({k: v["derived"] for k, v in doc.items() if k not in ("_how", "_meta")},
                     indent=1))
