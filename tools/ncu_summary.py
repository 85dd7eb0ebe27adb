"""Summarise an ncu report (raw page) into a compact JSON/markdown for profiles/ (dev tool)."""
import csv, io, json, subprocess, sys

KEYS = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
}
UNIT_SCALE = {"msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3,
              "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        k = {"kernel": d["Kernel Name"][:90]}
        for name, key in KEYS.items():
            if key in d and d[key] not in ("", "n/a"):
                v = float(d[key].replace(",", ""))
                if name == "time_ms":
                    v *= UNIT_SCALE.get(u[key], 1.0)
                elif name.endswith("bytes"):
                    v *= UNIT_SCALE.get(u[key], 1.0)
                k[name] = v
        stalls = [(kk.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(vv.replace(",", "")))
                  for kk, vv in d.items() if kk.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not kk.endswith("not_issued") and vv not in ("", "n/a")]
        tot = sum(v for _, v in stalls) or 1.0
        k["top_stalls_pct"] = {n: round(100 * v / tot, 1) for n, v in sorted(stalls, key=lambda x: -x[1])[:6]}
        res.append(k)
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1]), indent=1))
