"""Summarise an ncu report (ncu -i ... --page raw --csv) into profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_stage_v4 [--latest]

Writes <out>.json (per-kernel key metrics + stall breakdown) and, with
--latest, profiles/stage_kernel_latest.json (read by bench.py for the
roofline `traffic` field: dram bytes per launch of the stage kernel).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "smsp__inst_executed.sum": "warp_instructions",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")}
        for m, name in KEYS.items():
            if m in d and d[m]:
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                if u.get(m) == "Mbyte" or name.endswith("_MB"):
                    v = v if u.get(m) == "Mbyte" else v / 1e6 if u.get(m) == "byte" else v * 1e3 if u.get(m) == "Gbyte" else v
                if u.get(m) == "ms" and name == "duration_us":
                    v *= 1e3
                if u.get(m) == "ns" and name == "duration_us":
                    v /= 1e3
                k[name] = v
        st = [(float(v), h.split("stalled_")[1]) for h, v in d.items()
              if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and v]
        tot = sum(x for x, _ in st) or 1.0
        k["stalls_pct"] = {n: round(v / tot * 100, 1) for v, n in sorted(st, reverse=True)[:8]}
        if "dram_read_MB" in k and "dram_write_MB" in k:
            k["dram_bytes_per_launch"] = (k["dram_read_MB"] + k["dram_write_MB"]) * 1e6
        kernels.append(k)
    with open(out + ".json", "w") as fh:
        json.dump({"report": rep, "kernels": kernels}, fh, indent=1)
    if "--latest" in sys.argv:
        stage = [k for k in kernels if "stage_kernel" in k["kernel"]]
        if stage:
            with open("profiles/stage_kernel_latest.json", "w") as fh:
                json.dump(dict(stage[0], source=out + ".json"), fh, indent=1)
    for k in kernels:
        print(json.dumps(k))


if __name__ == "__main__":
    main()
