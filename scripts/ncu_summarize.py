"""Summarise the ncu outputs of scripts/gpu_profile.sh into profiles/ (tracked):
  profiles/<tag>_launches_<cfg>.csv   per kernel role: launches, mean gpu__time_duration, share of kernel time
  profiles/<tag>_ncu_full_<cfg>.csv   per captured launch (--set full): duration, DRAM bytes, tensor-pipe and
                                      memory throughput percentages, L2 hit rate
  profiles/ncu_traffic.json           dram__bytes_read.sum + dram__bytes_write.sum per launch by role (bench.py
                                      reads it for roofline.traffic)
usage: python scripts/ncu_summarize.py <tag> <cfg> [gpurun_out]"""
import csv, json, os, re, sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, cfg = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out")

# kernel template -> role (gemm_bf16_kernel<BN, EPI, AR, CG, CN>; Epi enum in cvr_kernels.cuh)
EPI = {0: "STORE", 1: "BIAS_RELU", 2: "CROSS", 3: "HEAD", 4: "BIAS", 5: "CROSS_F32", 6: "BIAS_ADD_F32", 7: "SUM_LN",
       8: "HEAD_PARTIAL", 9: "MASK", 10: "ATTN", 11: "ATTN_TC"}


def role(name):
    m = re.search(r"gemm_bf16_kernel<([\d, ]+)>", name)  # <BN, EPI, CG, EW>
    if m:
        bn, epi, cg = [int(x) for x in m.group(1).split(",")][:3]
        # role names of config 2 (for c6: BIAS_RELU = projection / mask hidden / MLP, MASK = mask blocks)
        r = {(0,): "gemm_xV", (2,): "gemm_tU_cross", (1,): "gemm_mlp_relu", (3,): "gemm_mlp_head",
             (9,): "gemm_mask_mul", (10,): "gemm_ens_qkv_attn", (5,): "gemm_tU_cross", (7,): "gemm_ens_ffn2_ln",
             (8,): "gemm_mlp_head", (11,): "gemm_ens_qkv_attn"}.get((epi,), f"gemm_{EPI.get(epi, epi)}")
        return f"{r} [BN={bn}{' pair' if cg == 2 else ''}]"
    if "ffn_fused" in name:
        return "gemm_ens_ffn_fused"
    for k in ("embed_bag", "dense_f32", "unpack", "mha64", "head_finalize", "set_call"):
        if k in name:
            return k
    return name[:60]


def rows(path):
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    return list(csv.reader(lines))


# ---- launch list
L = rows(os.path.join(src, f"launches_{cfg}.csv"))
hdr = L[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = OrderedDict()
for r in L[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    k = role(r[ki])
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) / 1e3
tot = sum(v[1] for v in agg.values())
out = os.path.join(ROOT, "profiles", f"{tag}_launches_{cfg}.csv")
with open(out, "w") as f:
    f.write("# ncu launch list: gpu__time_duration.sum --clock-control none (serialised, cold cache: compare SHARES)\n")
    f.write(f"# command: python bench.py --config {cfg} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-serving (scripts/gpu_profile.sh)\n")
    f.write("kernel, launches, avg_us, share_of_kernel_time\n")
    for k, (n, t) in agg.items():
        f.write(f"{k}, {n}, {t / n:.2f}, {t / tot:.3f}\n")
print(open(out).read())

# ---- full capture
F = rows(os.path.join(src, f"prof_full_{cfg}_raw.csv"))
hdr, units, data = F[0], F[1], F[2:]
col = {h: i for i, h in enumerate(hdr)}
want = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB", None), ("dram__bytes_write.sum", "MB", None),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct", 1),
        ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "tc_smem_read_pct", 1),
        ("lts__t_sector_hit_rate.pct", "l2_hit_pct", 1)]


def val(r, name, unit_scale):
    if name not in col:
        return None
    v = r[col[name]].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    u = units[col[name]]
    if unit_scale is None:  # bytes -> MB
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) / 1e6
    elif name == "gpu__time_duration.sum":
        x *= {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3}.get(u, 1e-3)
    return x


out = os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{cfg}.csv")
traffic = {}
with open(out, "w") as f:
    f.write("# ncu --set full --clock-control none (replayed, caches flushed between passes: L2-resident activations\n")
    f.write("# count as DRAM traffic); one step's kernels from the middle of the run (scripts/gpu_profile.sh)\n")
    f.write("kernel, duration_us, dram_read_MB, dram_write_MB, dram_pct, compute_memory_pct, tc_smem_read_pct, l2_hit_pct\n")
    for r in data:
        k = role(r[col["Kernel Name"]])
        vals = [val(r, n, s) for n, _, s in want]
        f.write(k + ", " + ", ".join("" if v is None else f"{v:.2f}" for v in vals) + "\n")
        base = k.split(" [")[0]
        if vals[1] is not None and vals[2] is not None:
            traffic.setdefault(base, []).append((vals[1] + vals[2]) * 1e6)
print(open(out).read())
tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
old = json.load(open(tp)) if os.path.exists(tp) else {}
if not isinstance(old.get(cfg, {}), dict) or "_note" not in old or "by_config" not in old.get("_format", ""):
    old = {"_format": "by_config: {config: {kernel role: bytes per launch}}"}
old[cfg] = {("embed_bag_pool" if k == "embed_bag" else k): sum(v) / len(v) for k, v in traffic.items()}
old["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over the captured launches of the "
                "role; ncu --set full replays with caches flushed (cold L2), so L2-resident activations count as DRAM "
                "traffic here (tag %s)" % tag)
json.dump(old, open(tp, "w"), indent=1)
