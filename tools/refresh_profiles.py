"""Copy a round_gpu.sh run (suffix, e.g. final3) into profiles/: bench line, GPU test log, smoke log, launch
list + summary, ncu summary and DRAM traffic of the 2D RAS apply (profiles/ncu_traffic.json feeds bench.py)."""
import collections, csv, json, os, shutil, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
suf = sys.argv[1]
shutil.copy(os.path.join(G, f"bench_{suf}.log"), os.path.join(P, "r01_bench_final.log"))
shutil.copy(os.path.join(G, f"gpu_tests_{suf}.log"), os.path.join(P, "r01_gpu_tests_final.log"))
shutil.copy(os.path.join(G, f"smoke_{suf}.log"), os.path.join(P, "r01_smoke_final.log"))
shutil.copy(os.path.join(G, f"launches_{suf}.csv"), os.path.join(P, "r01_launches_final.csv"))

rows = list(csv.reader(open(os.path.join(G, "r2_raw.csv"))))
h, units, r = rows[0], rows[1], rows[2]
g = lambda n: r[h.index(n)]
rd = float(g("dram__bytes_read.sum")) * 1e6
wr = float(g("dram__bytes_write.sum")) * 1e6
kname = g("Kernel Name")
json.dump({"_source": "ncu --set full --clock-control none -k regex:k_apply -s 2 -c 1 python tools/time_pc.py (CFG=2) -- "
                      "tools/ncu_r2.sh; summary profiles/r01_ncu_r2_apply_summary.txt",
           "ras_apply": {"kernel": "nks::r2::" + kname, "grid": [512, 512], "dram_bytes_per_launch": int(rd + wr),
                         "dram_read": int(rd), "dram_write": int(wr),
                         "duration_us_cold_serialised": float(g("gpu__time_duration.sum"))}},
          open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
lines = [f"ncu --set full, r2::{kname} (2D RAS apply, final round-1 version), config 2 (512^2, 4x4 boxes, delta 2), "
         "tools/ncu_r2.sh"]
lines += [f"    {k:70s} {units[h.index(k)]:>12s} {g(k)}" for k in keys if k in h]
steps = 96 * 352
lines.append(f"per CTA-step (96 CTAs x 2 x 176 steps): shared wavefronts "
             f"{float(g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')) / steps:.0f}, warp instructions "
             f"{float(g('smsp__inst_executed.sum')) / steps:.0f}")
lines.append(f"DRAM {rd / 1e6:.1f} MB read + {wr / 1e6:.1f} MB written per launch = {(rd + wr) / 1e6:.1f} MB "
             "(algorithmic 481.2 MB)")
ks = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
st = sorted(((float(g(k) or 0), k) for k in ks), reverse=True)[:8]
lines.append("top stall samples: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {int(v)}"
                                               for v, k in st))
open(os.path.join(P, "r01_ncu_r2_apply_summary.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

rows = list(csv.reader(l for l in open(os.path.join(G, f"launches_{suf}.csv")) if not l.startswith("==")))
h = rows[0]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
t, n = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    t[r[ik][:60]] += float(r[iv].replace(",", ""))
    n[r[ik][:60]] += 1
tot = sum(t.values())
out = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 3000: python bench.py --steps 1 --warmup 3 "
       "(first 3000 launches; cold-cache, serialised per-launch times)"]
out += [f"{v / tot * 100:6.2f}%  {v / 1e3:10.1f} us  {n[k]:6d} launches  {k}" for k, v in t.most_common(15)]
open(os.path.join(P, "r01_launches_final_summary.txt"), "w").write("\n".join(out) + "\n")
print(out[1])
