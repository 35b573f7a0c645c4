"""Summary of one `ncu --set full` capture of an onesweep pass (what
profiles/r02_onesweep_traffic_cfg3.json holds): duration, DRAM bytes against
the algorithmic bytes, L1 data-pipe and issue utilisation, shared-memory
wavefronts per 32 keys, top stalls.

  python tools/ncu_traffic_summary.py gpurun_out/r02e_onesweep_cfg3.ncu-rep N_KEYS KEY_BYTES > profiles/...json
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, n, kb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}

    def val(name, scale=None):
        v = float(vals[col[name]].replace(",", ""))
        u = units[col[name]]
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3,
                "ns": 1e-6, "s": 1e3}.get(u, 1)
        return v * mult

    alg = 2 * kb * n
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    rows32 = n / 32
    stalls = {h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]:
              float(vals[i]) for h, i in col.items()
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
    top = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    out = {
        "source": f"ncu --set full --clock-control none, {rep.split('/')[-1]} (tools/round_profile.sh)",
        "kernel": vals[col["Kernel Name"]].split("(")[0],
        "workload": f"{n} keys of {kb} bytes, one digit pass",
        "gpu__time_duration_ms": val("gpu__time_duration.sum"),
        "dram__bytes_read": rd, "dram__bytes_write": wr,
        "algorithmic_bytes_per_launch": alg,
        "traffic_bytes_per_launch": rd + wr,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "smsp__issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "l1tex_data_pipe_lsu_wavefronts_pct": val("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "shared_wavefronts_per_32_keys": {
            op: val(f"l1tex__data_pipe_lsu_wavefronts_mem_shared_op_{op}.sum") / rows32
            for op in ("atom", "ld", "st")},
        "stall_per_issue_top": top,
        "registers_per_thread": int(val("launch__registers_per_thread")),
        "grid": int(val("launch__grid_size")), "block": int(val("launch__block_size")),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
