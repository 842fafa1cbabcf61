"""Write profiles/<round>_ncu_summary.md and profiles/force_traffic.json from
the outputs of tools/refresh_profiles.sh (gpurun_out/): the bench line, the
ncu launch list and the --set full captures.
Usage: python tools/write_summary.py [round-tag, default r02]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def summary(rep):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                         capture_output=True, text=True, check=True).stdout
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


b = json.loads(open(os.path.join(G, "bench.json")).read().strip().splitlines()[-1])
rf = b["roofline"]
cols = ["time_ms", "dram_read_MB", "dram_write_MB", "dram_pct", "l1_pct", "l2_pct", "l1_hit",
        "issue_pct", "warps_active_pct", "fma_pct", "regs", "inst"]
caps = {}
for name in ("step_full", "sph_rates_full", "dem_step_full"):
    for r in summary(os.path.join(G, name + ".ncu-rep")):
        k = r["kernel"].replace("void ", "").replace("unnamed>::", "")
        caps.setdefault(k, []).append(r)
lj = next(v for k, v in caps.items() if k.startswith("k_lj_step<0"))
traffic = sum(r["dram_read_MB"] + r["dram_write_MB"] for r in lj) / len(lj) * 1e6
nbar_cap = None
for line in open(os.path.join(G, "step_full.log")):
    if line.startswith("{") and "mean_row" in line:
        nbar_cap = json.loads(line)["mean_row"]
json.dump({"kernel": "k_lj_step<0> (force sweep + fused VV)", "bytes_per_launch": traffic,
           "nbar_at_capture": nbar_cap,
           "source": f"profiles/{TAG}_ncu_summary.md (ncu --set full, tools/prof_step.py cfg2 "
                     "liquid phase, mean over the captured launches of dram__bytes_read.sum + "
                     "dram__bytes_write.sum); bench.py scales it by (4 nbar + 64) / (4 "
                     "nbar_at_capture + 64) to the bench run's mean row"},
          open(os.path.join(P, "force_traffic.json"), "w"), indent=1)
launches = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_launches.py"),
                           os.path.join(G, "launches.csv")], capture_output=True, text=True,
                          check=True).stdout
L = []
L.append("# Round %s profile summary (B200, sm_100a)\n" % TAG[1:])
L.append("Produced by `tools/refresh_profiles.sh` (one gpurun call) and `tools/write_summary.py`.\n")
L.append("Bench line (`python bench.py`, defaults: %d timed steps after %d warm-up): "
         "profiles/%s_bench.json\n" % (b["steps"], b["warmup"], TAG))
L.append("- value %.4g particle-updates/s, %.1f us/step, %d rebuilds in %d steps, mean row %.2f"
         % (b["value"], 1e3 * b["ms_per_step"], b["config"]["rebuilds"], b["steps"],
            b["config"]["mean_row"]))
L.append("- dominant kernel %s: %.1f us/launch (CUDA events in the step graph), %.0f GB/s "
         "algorithmic = %.3f of measured HBM %.1f GB/s; share of step %.2f; DRAM traffic "
         "%.0f MB/launch vs %.0f MB algorithmic (measured-DRAM fraction %.3f)"
         % (rf["kernel"], 1e3 * rf["kernel_ms"], rf["achieved"], rf["frac"], rf["peak"],
            rf["kernel_share_of_step"], traffic / 1e6, rf["alg_bytes_per_launch"] / 1e6,
            traffic / (rf["kernel_ms"] * 1e-3) / 1e9 / rf["peak"]))
L.append("- e2e (pinned host in/out through the C-ABI): %.4g PU/s" % b["e2e"]["value"])
L.append("- SPH pass (cfg4, %d particles): %.2f ms; SPH time stepping (pm_sph_run): %.3f ms/step "
         "= %.4g particle-steps/s" % (b["sph"]["n_particles"], b["sph"]["pass_ms"],
                                      b["sph"]["run"]["ms_per_step"], b["sph"]["run"]["value"]))
L.append("- DEM avalanche (%d grains, pm_dem_run): %.4f ms/step = %.4g particle-steps/s"
         % (b["dem"]["n_particles"], b["dem"]["ms_per_step"], b["dem"]["value"]))
cb = b.get("cpu_baseline") or {}
if cb:
    L.append("- CPU oracle baseline: %.0f PU/s on %d host cores (%s)"
             % (cb["value"], cb["cores"], cb["sample"]))
L.append("- clocks during the timed region: %s\n" % b["clocks"])
L.append("## ncu --set full captures\n")
L.append("k_lj_step / k_verlet: `tools/prof_step.py --steps 200` (cfg2, non-graph), launches "
         "20-31; k_sph_rates: `tools/exp_sph_rate.py` (cfg4 stepping), launch 51; k_dem_step: "
         "`tools/dem_prof.py 300 50` (avalanche), launch 321.  Means over the captured launches.\n")
L.append("| kernel | launches | " + " | ".join(cols) + " |")
L.append("|---|---|" + "---|" * len(cols))
for k, rs in caps.items():
    m = {c: sum(r[c] for r in rs) / len(rs) for c in cols}
    L.append("| %s | %d | " % (k, len(rs)) + " | ".join(
        ("%.4g" % m[c]) if c != "inst" else ("%.4g" % m[c]) for c in cols) + " |")
L.append("")
L.append("k_lj_step: the L1 data pipe is busy with the scattered float4 gathers, but it is not "
         "the bound alone: the gather-order microbenchmark (tools/micro/gather_order.cu, "
         "DESIGN.md §11) cuts L1 wavefronts by 21%% for a 2%% gain, and without any memory stall "
         "(L1-hit gathers, no index stream) the same loop still takes 0.11 ms -- instruction "
         "issue plus gather latency (long scoreboard).  k_verlet_st (staged build): coalesced candidate stages, "
         "paired fp32 tests, predicated appends into 16-bit shared-memory rows, full-line "
         "flushes (no write amplification).  k_sph_rates / k_dem_step as in round 1.\n")
L.append("## Launch list (`PM_USE_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control "
         "none` of `python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-extras`: the "
         "cfg2 step alone; cold-cache, serialised: compare shares)\n")
L.append(launches)
open(os.path.join(P, f"{TAG}_ncu_summary.md"), "w").write("\n".join(L))
print("\n".join(L[:12]))
