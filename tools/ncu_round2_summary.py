"""Summarise the round-2 evidence (tools/r2_profile.sh TAG outputs) into
profiles/r2_final_ncu.json and per-launch DRAM traffic into
profiles/ncu_traffic.json.  usage: python tools/ncu_round2_summary.py [TAG]"""
import csv, io, json, os, subprocess, sys
T = sys.argv[1] if len(sys.argv) > 1 else "r2f"
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum" and "kapsm" in d["Kernel Name"]:
                out.append((d["Kernel Name"].split("(")[0].replace("void ", ""),
                            float(d["Metric Value"]) / 1e3))
    return out


def full(path, names):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    R = list(csv.reader(io.StringIO(raw)))
    H, U = R[0], R[1]
    out = {}
    for i, r in enumerate(R[2:]):
        key = names[i] if i < len(names) else r[H.index("Kernel Name")].split("(")[0]
        d = {k: r[H.index(k)] + (" " + U[H.index(k)] if U[H.index(k)] else "") for k in KEYS if k in H}
        b = sum(float(r[H.index(k)]) * UNIT.get(U[H.index(k)], 1)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        d["dram_bytes_per_launch"] = int(b)
        out[key] = d
    return out


tp_names = ["detect_screen_tc", "band_rows", "pilot_screen_tc", "apsm_train_tp", "detect_finish"]
lat_names = ["pilot_gram", "detect_screen_tc", "apsm_train", "detect_finish"]
res = {"what": ("round-2 evidence (tools/r2_profile.sh " + T + "): ncu launch lists (cold, "
                "serialised) and --set full per kernel of one 1184-frame throughput pipeline "
                "launch and of one single-frame latency pipeline launch (tools/tp_launches.py), "
                "and the band trainer of the single-frame C4 full band / C3 n2048 W64 configs"),
       "throughput_1184": {"launches_us": launches(f"gpurun_out/{T}_launches_tp.csv"),
                           "full": full(f"gpurun_out/{T}_full_tp.ncu-rep", tp_names)},
       "latency_1": {"launches_us": launches(f"gpurun_out/{T}_launches_lat.csv"),
                     "full": full(f"gpurun_out/{T}_full_lat.ncu-rep", lat_names)}}
for key, rep in (("c4_full_band_trainer", f"gpurun_out/{T}_full_c4fb.ncu-rep"),
                 ("c3_n2048_w64_trainer", f"gpurun_out/{T}_full_c3.ncu-rep")):
    if os.path.exists(rep):
        res[key] = full(rep, ["apsm_train_tpl"])
json.dump(res, open("profiles/r2_final_ncu.json", "w"), indent=1)
tr = json.load(open("profiles/ncu_traffic.json"))
for k, v in res["throughput_1184"]["full"].items():
    tr[f"{k}_batch_bytes_per_launch"] = v["dram_bytes_per_launch"]
tr["batch_frames"] = 1184
for k, v in res["latency_1"]["full"].items():
    tr[f"{k}_bytes_per_launch"] = v["dram_bytes_per_launch"]
tr["source_batch"] = "profiles/r2_final_ncu.json (throughput_1184)"
tr["source"] = "profiles/r2_final_ncu.json (latency_1; ncu flushes L2 between replays)"
json.dump(tr, open("profiles/ncu_traffic.json", "w"), indent=1)
for sec in ("throughput_1184", "latency_1"):
    print(sec, res[sec]["launches_us"])
    for k, v in res[sec]["full"].items():
        print("  ", k, v["gpu__time_duration.sum"], v["dram_bytes_per_launch"] / 1e6, "MB",
              v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              v.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"))
