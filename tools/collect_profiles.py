"""Copy one GPU evidence pass (tools/gpu_round.sh TAG) from gpurun_out/ into profiles/<round>/:
bench lines, launch lists + summaries, the ncu --set full raw page + summary + the counters the
roofline discussion uses, and the per-kernel DRAM traffic (profiles/ncu_traffic.json).

    python tools/collect_profiles.py r02c r02
"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

tag, rnd = sys.argv[1], sys.argv[2]
root = Path(__file__).resolve().parents[1]
src, dst = root / "gpurun_out", root / "profiles" / rnd
dst.mkdir(parents=True, exist_ok=True)


def run(*cmd):
    return subprocess.run(list(cmd), capture_output=True, text=True, cwd=root).stdout


def copy(name, out=None):
    if (src / name).exists():
        shutil.copy(src / name, dst / (out or name))
        return True
    return False


copy(f"bench_{tag}.json", f"bench_{rnd}.json")
copy(f"bench_ref_{tag}.json", f"bench_ref_{rnd}.json")
for n in ("pytest_gpu.log", "smoke.log", "smi.txt"):
    copy(n)
copy(f"small_profile_{tag}.txt", f"small_profile_{rnd}.txt")
for n in ("early_iters.txt", "cold_phases.txt"):
    copy(n)
summ = []
for name, label in ((f"launches_{tag}.csv", "bench.py --steps 20 --warmup 5 (setup + iterations 1..30), config 4"),
                    (f"launches_steady_{tag}.csv", "config 4, ~iterations 200..216 (steady state)")):
    if copy(name, name.replace(tag, rnd)):
        summ.append(run(sys.executable, "tools/launch_summary.py", str(src / name), label))
for c in range(4):
    name = f"launches_cfg{c}_{tag}.csv"
    if copy(name, name.replace(tag, rnd)):
        summ.append(run(sys.executable, "tools/launch_summary.py", str(src / name),
                        f"config {c}, hot kernels of ~iterations 30..45 (tools/profile_run.py --iters 80)"))
(dst / "launches_summary.txt").write_text(
    "# ncu --metrics gpu__time_duration.sum --clock-control none (cold caches, serialised): shares, not absolutes\n\n"
    + "\n\n".join(summ))

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
        "sm__cycles_active.avg", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__registers_per_thread", "launch__waves_per_multiprocessor",
        "sm__inst_executed.sum", "smsp__inst_executed_pipe_fp64.sum", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for rep, out in ((f"full_{tag}.ncu-rep", "ncu_full"), ("full_cold.ncu-rep", "ncu_cold")):
    if not (src / rep).exists():
        continue
    raw = run("ncu", "-i", str(src / rep), "--page", "raw", "--csv")
    (dst / f"{out}_raw.csv").write_text(raw)
    (dst / f"{out}_summary.txt").write_text(run(sys.executable, "tools/ncu_summary.py", str(src / rep)))
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    traffic = {}
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        kname = d["Kernel Name"].split("(")[0].replace("void ", "")
        lines.append(f"== [{d['ID']}] {kname}")
        for w in WANT:
            for h, u in zip(hdr, units):
                if h == w and d.get(h):
                    lines.append(f"   {h:70s} {d[h]} {u}")
        try:
            by = float(d["dram__bytes_read.sum"].replace(",", "")) + float(d["dram__bytes_write.sum"].replace(",", ""))
            ur, uw = units[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            by = (float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(ur, 1)
                  + float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(uw, 1))
            base = kname.split("<")[0].replace("hsde::", "")
            traffic.setdefault(base, []).append(by)
        except (KeyError, ValueError):
            pass
    (dst / f"{out}_counters.txt").write_text("\n".join(lines) + "\n")
    if out == "ncu_full" and traffic:
        per = {k: int(max(v)) for k, v in traffic.items()}
        slots = {"k_rhs": per.get("k_rhs"), "k_spmv_seg": sum(per.get(k, 0) for k in ("k_pair_sum", "k_spmv_half", "k_rowsum_tiles")),
                 "k_schur": per.get("k_schur"), "k_ua": per.get("k_ua_half"), "k_scalars": per.get("k_scalars"),
                 "k_cone_cta": per.get("k_cone_split"), "k_xupd": per.get("k_xupd")}
        slots["_per_kernel"] = per
        slots["_source"] = (f"ncu --set full, config 4, iteration ~200, dram__bytes_read.sum + dram__bytes_write.sum per launch "
                            f"(profiles/{rnd}/ncu_full_raw.csv, {rep})")
        (root / "profiles" / "ncu_traffic.json").write_text(json.dumps(slots, indent=1))
print("collected into", dst)
