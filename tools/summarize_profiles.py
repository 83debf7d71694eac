"""Summarise a round's ncu captures (gpurun_out/launches_<R>.csv and
gpurun_out/prof_<R>.ncu-rep) into tracked files under profiles/:

  profiles/<R>_launches.csv       the launch list (copied)
  profiles/<R>_launch_shares.md   per-kernel device time share of one step
  profiles/<R>_ncu_full.json      per-kernel duration, DRAM bytes, utilisation
  profiles/<R>_ncu_full.md        the same as a table
  profiles/traffic.json           DRAM bytes per launch per bench op (read by
                                  bench.py for roofline.traffic)

    python tools/summarize_profiles.py r1
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

OP_OF_KERNEL = [  # kernel name prefix -> bench op
    ("softmax_fwd_vec_kernel", "softmax_dropout_fwd"),
    ("softmax_bwd_vec_kernel", "attn_probs_bwd"),
    ("gelu_fwd_vec_kernel", "gelu_fwd"),
    ("gelu_fwd8_kernel", "gelu_fwd"),
    ("gelu_bwd_fast_kernel", "gelu_bwd"),
    ("ln_fwd_vec_kernel", "layernorm_fwd"),
    ("ln_fwd_warp_kernel", "layernorm_fwd"),
    ("ln_bwd_vec_kernel<256, 1, 1>", "dropout_add_layernorm_bwd"),
    ("dal_fwd_warp_kernel", "dropout_add_layernorm_fwd"),
    ("ln_bwd_vec_kernel", "layernorm_bwd"),
    ("ln_param_reduce_kernel", "layernorm_bwd"),
    ("ln_param_reduce8_kernel", "layernorm_bwd"),
    ("dropout_fwd_vec_kernel<1>", "dropout_fwd"),
    ("dropout_fwd8_kernel<1", "dropout_fwd"),
    ("dropout_fwd8_kernel<0", "dropout_bwd"),
    ("dropout_fwd_vec_kernel<0>", "dropout_bwd"),
]


def op_of(kernel):
    k = kernel.split("::")[-1] if "::" in kernel else kernel
    for pre, op in OP_OF_KERNEL:
        if pre in kernel:
            return op
    return None


def main(r):
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    out = os.path.join(ROOT, "gpurun_out")
    lcsv = os.path.join(out, f"launches_{r}.csv")
    if os.path.exists(lcsv):
        shutil.copy(lcsv, os.path.join(prof, f"{r}_launches.csv"))
        rows = [x for x in csv.reader(open(lcsv)) if len(x) > 10]
        hdr = rows[0]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        per = {}
        for x in rows[1:]:
            if x[mi] != "gpu__time_duration.sum":
                continue
            per.setdefault(x[ki], []).append(float(x[vi].replace(",", "")))
        tot = sum(sum(v) for v in per.values())
        lines = [f"# {r}: launch list of `bench.py --steps 2 --warmup 1` under ncu",
                 "", "Cold-cache, serialised launches: compare shares, not absolutes.", "",
                 "| kernel | launches | mean us | share of captured time |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | "
                         f"{sum(v)/tot:.3f} |")
        open(os.path.join(prof, f"{r}_launch_shares.md"), "w").write("\n".join(lines) + "\n")
    rep = os.path.join(out, f"prof_{r}.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        tmp = os.path.join(out, f"raw_{r}.csv")
        open(tmp, "w").write(raw)
        recs = ncu_summary.main(tmp)
        json.dump(recs, open(os.path.join(prof, f"{r}_ncu_full.json"), "w"), indent=1)
        lines = [f"# {r}: ncu --set full, bench shapes (BERT-large layer, B=64; "
                 "tools/profile_ops.py: the fused chain's ops, then the unfused LN/dropout ops, "
                 "then configs[0..2])", "",
                 "| kernel | us | DRAM read MB | DRAM write MB | DRAM % (ncu peak) | issue % | "
                 "warps active % | regs |", "|---|---|---|---|---|---|---|---|"]
        traffic = {}
        for d in recs:
            lines.append(f"| `{d['kernel'][:60]}` | {d.get('duration_us', 0):.1f} | "
                         f"{d.get('dram_read_B', 0)/1e6:.1f} | {d.get('dram_write_B', 0)/1e6:.1f} | "
                         f"{d.get('dram_pct', 0):.1f} | {d.get('issue_active_pct', 0):.1f} | "
                         f"{d.get('warps_active_pct', 0):.1f} | {d.get('regs', 0):.0f} |")
            op = op_of(d["kernel"])
            if op and op not in traffic:
                traffic[op] = int(d.get("dram_read_B", 0) + d.get("dram_write_B", 0))
        open(os.path.join(prof, f"{r}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
        json.dump(traffic, open(os.path.join(prof, "traffic.json"), "w"), indent=1)
    print("profiles written for", r)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
