"""Summarise gpurun_out ncu reports into profiles/ (tracked)."""
import csv
import json
import os
import sys
import collections

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
# on the GPU box: PROFILES_OUT=gpurun_out/profiles_out (merged back), then copied
P = os.environ.get("PROFILES_OUT", os.path.join(ROOT, "profiles"))
os.makedirs(P, exist_ok=True)
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}


def kernel_entry(path):
    d = summary(path)[0]
    val = lambda m: float(d[m][0]) * UNIT.get(d[m][1], 1)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur = val("gpu__time_duration.sum")
    return {"kernel": d["kernel"], "dram_bytes": int(rd + wr), "dram_read": int(rd),
            "dram_write": int(wr), "duration_us_ncu": round(dur * 1e6, 1),
            "dram_gbs_ncu": round((rd + wr) / dur / 1e9, 1),
            "dram_pct_of_theoretical": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
            "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
            "registers": int(float(d["launch__registers_per_thread"][0])),
            "l1_hit_pct": float(d["l1tex__t_sector_hit_rate.pct"][0]),
            "l2_hit_pct": float(d["lts__t_sector_hit_rate.pct"][0])}


def lib_sha16():
    import hashlib
    with open(os.path.join(ROOT, "paper_2306_17801_b200", "lib", "librvk.so"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def build_id():
    sys.path.insert(0, ROOT)
    from paper_2306_17801_b200 import rvk
    return rvk.lib().rvk_build_id().decode()


def main(tag="r02"):
    # the captures in gpurun_out/ must come from the library now in the tree
    # (scripts/gpu_profiles.sh runs on the snapshot of this tree)
    out = {"_note": f"{tag}: ncu --set full --clock-control none, one launch each "
                    "(serialised, after 4 warm launches); per-launch DRAM bytes = traffic",
           "lib_sha16": lib_sha16(), "build_id": build_id()}
    for cfg, files in {"7pt256": {"k1": "prof_k1", "k2": "prof_k2"},
                       "7pt768": {"k1": "prof_k1_768"},
                       "27pt256": {"k1": "prof_k1_27pt"}, "9pt4096": {"k1": "prof_k1_9pt"},
                       "7pt256_matrix_free": {"k1": "prof_mf"},
                       "27pt256_matrix_free": {"k1": "prof_mf_27pt"},
                       "5pt768_grid_l2": {"solve": "prof_gridl2_768"}}.items():
        for k, f in files.items():
            path = os.path.join(G, f + ".ncu-rep")
            if os.path.exists(path):
                out.setdefault(cfg, {})[k] = kernel_entry(path)
    # one whole P = 1 row-shard solve (the N > 1 bench line's per-GPU traffic):
    # every kernel inside the NVTX range dcg.loopback_solve
    sp = os.path.join(G, "shard_solve_dram.csv")
    if os.path.exists(sp):
        txt = open(sp).read().splitlines()
        hdr = next((r for r in csv.reader(txt) if r and r[0] == "ID"), None)
        if hdr:
            im, iv = hdr.index("Metric Name"), hdr.index("Metric Value")
            tot = collections.defaultdict(float)
            ids = set()
            for r in csv.reader(txt):
                if len(r) > iv and r[0].isdigit():
                    tot[r[im]] += float(r[iv])
                    ids.add(r[0])
            rd, wr = tot["dram__bytes_read.sum"], tot["dram__bytes_write.sum"]
            out["7pt256_shard"] = {"solve": {
                "kernels": len(ids), "dram_bytes": int(rd + wr), "dram_read": int(rd),
                "dram_write": int(wr), "kernel_time_us_ncu": round(tot["gpu__time_duration.sum"] / 1e3, 1),
                "capture": "ncu --nvtx --nvtx-include dcg.loopback_solve/ (P = 1 shard, 256^3 7-point)"}}
    with open(os.path.join(P, "ncu_summary.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    # launch list shares
    rows = [r for r in csv.reader(open(os.path.join(G, "launches.csv"))) if len(r) > 10 and r[0].isdigit()]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r[4].split("(")[0]
        tot[name] += float(r[-1]) / 1000
        cnt[name] += 1
    T = sum(tot.values())
    with open(os.path.join(P, f"{tag}_launch_shares_7pt256.txt"), "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum launch list, 2 solves of 3D 7-pt 256^3\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            fh.write(f"{k:45s} n={cnt[k]:3d} total={tot[k]:9.1f} us avg={tot[k]/cnt[k]:8.1f} us "
                     f"share={tot[k]/T:6.1%}\n")
    os.replace(os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches_7pt256.csv")) \
        if os.path.exists(os.path.join(G, "launches.csv")) else None
    print(open(os.path.join(P, f"{tag}_launch_shares_7pt256.txt")).read())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*(sys.argv[1:]))
