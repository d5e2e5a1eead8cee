"""Per-kernel roofline table from `ncu --set full` captures of one c3 critic
update, one policy update and one actor step + ingest (tools/ncu_all.sh):
algorithmic work (FLOP for the tensor-core GEMMs, bytes for the HBM-bound
kernels, SURVEY §8(d) / App. C formulas) / ncu duration, as a fraction of
the measured peaks (cuBLAS TF32 8192^3 from bench.py; HBM copy bandwidth
from MEASURED_PEAKS.json), with the measured DRAM traffic and tensor-pipe
utilisation beside it.  For a GEMM the binding roof is the larger of
FLOP / TF32 peak and operand bytes / HBM peak (operand bytes count A, B and
D once per group, so inputs shared by two groups count twice -- a generous
HBM roof).  ncu durations are cold-cache and serialised, so the
fractions are lower bounds of the in-graph ones.

  python tools/roofline_table.py [dir] > profiles/r1_roofline_table.md

[dir] holds all_{critic,policy,actor}_raw.csv (tools/ncu_all.sh); without it
the trimmed copies committed as profiles/r1_ncu_{critic,policy,actor}.csv
are read.
"""
import csv
import json
import sys
from pathlib import Path

D, A, H, B, N = 211, 20, 512, 8192, 16384
K0, Kp, Dp = D + A, 232, 212
TF32_PEAK = 770e12      # cuBLAS TF32 8192^3, measured in bench.py (roofline.peak)
HBM_PEAK = None         # from MEASURED_PEAKS.json


def gemm(M, Nn, K, groups=1):
    # FLOP, plus the operand bytes (A, B and D once per group, fp32) so the
    # binding roof is max(FLOP / TF32 peak, bytes / HBM peak): the thin
    # 512->20 heads are bounded by reading their activations, not by MMA.
    return ("tensor", 2.0 * M * Nn * K * groups, 4.0 * groups * (M * K + K * Nn + M * Nn))


def hbm(nbytes):
    return ("hbm", float(nbytes))


P_CRIT = (K0 * H + H) + 2 * (H * H + H) + (H + 1)
P_POL = (D * H + H) + 2 * (H * H + H) + (H * A + A)
CRITIC = [
    ("replay sample + normalise (gather)", "replay_sample", hbm(2 * B * (2 * D + A + 2) * 4)),
    ("target policy L0", "Hidden", gemm(B, H, D)),
    ("target policy L1", "Hidden", gemm(B, H, H)),
    ("target policy L2", "Hidden", gemm(B, H, H)),
    ("target policy head (split-K)", "Partial", gemm(B, A, H)),
    ("target policy head finish", "finish", hbm(4 * B * A * 4 + B * A * 4)),
    ("4-group critics L0 (q1',q2',q1,q2)", "Hidden", gemm(B, H, K0, 4)),
    ("4-group critics L1", "Hidden", gemm(B, H, H, 4)),
    ("4-group critics L2 (+512->1 head dots)", "Hidden", gemm(B, H, H, 4)),
    ("TD target + loss + upstream", "critic_loss", hbm(2 * 2 * 4 * B * 4 + 6 * B * 4)),
    ("value-head backward", "head_backward", hbm(2 * 2 * B * H * 4)),
    ("wgrad L2 (split-K)", "Partial", gemm(H, H, B, 2)),
    ("dgrad L2 (+mask, bias sums)", "DgradMask", gemm(B, H, H, 2)),
    ("wgrad L1 (split-K)", "Partial", gemm(H, H, B, 2)),
    ("dgrad L1 (+mask, bias sums)", "DgradMask", gemm(B, H, H, 2)),
    ("wgrad L0 (split-K)", "Partial", gemm(K0, H, B, 2)),
    ("split-K reduction + fp64 norm + clip scale", "finalize",
     hbm(2 * 4 * (18 * K0 * H + 9 * H * H * 2) + 2 * P_CRIT * 4)),
    ("clip + Adam + Polyak (2 critics)", "adam", hbm(2 * P_CRIT * 36)),
]
POLICY = [
    ("state sample + normalise", "state_sample", hbm(2 * B * D * 4)),
    ("policy L0", "Hidden", gemm(B, H, D)),
    ("policy L1", "Hidden", gemm(B, H, H)),
    ("policy L2", "Hidden", gemm(B, H, H)),
    ("policy head (split-K)", "Partial", gemm(B, A, H)),
    ("policy head finish (+tanh out)", "finish", hbm(4 * B * A * 4 + 2 * B * A * 4)),
    ("twin critics L0", "Hidden", gemm(B, H, K0, 2)),
    ("twin critics L1", "Hidden", gemm(B, H, H, 2)),
    ("twin critics L2 (+head dots)", "Hidden", gemm(B, H, H, 2)),
    ("min-critic pick", "actor_pick", hbm(2 * 4 * B * 4 + 2 * B * 4)),
    ("value-head input gradient", "head_input_grad", hbm(2 * B * H * 4)),
    ("critic dgrad L2", "DgradMask", gemm(B, H, H, 2)),
    ("critic dgrad L1", "DgradMask", gemm(B, H, H, 2)),
    ("critic dgrad L0 (action columns)", "Store", gemm(B, A, H, 2)),
    ("policy head backward", "policy_head_backward", hbm(4 * B * A * 4)),
    ("policy head wgrad", "Partial", gemm(H, A, B)),
    ("policy head dgrad", "DgradMask", gemm(B, H, A)),
    ("policy wgrad L2", "Partial", gemm(H, H, B)),
    ("policy dgrad L2", "DgradMask", gemm(B, H, H)),
    ("policy wgrad L1", "Partial", gemm(H, H, B)),
    ("policy dgrad L1", "DgradMask", gemm(B, H, H)),
    ("policy wgrad L0", "Partial", gemm(D, H, B)),
    ("split-K reduction + norm", "finalize", hbm(4 * (18 * D * H + 9 * H * H * 2) + P_POL * 4)),
    ("clip + Adam (policy)", "adam", hbm(P_POL * 32)),
]
ACTOR = [  # (label, name key, work, ncu row index)
    ("policy L0 (16384 envs)", "Hidden", gemm(N, H, D), 9),
    ("policy L1", "Hidden", gemm(N, H, H), 10),
    ("policy L2", "Hidden", gemm(N, H, H), 11),
    ("policy head + squash + mixed noise", "PolicyHead", gemm(N, A, H), 1),
    ("running-normalizer update (fp64)", "norm_update", hbm(N * D * 4), 2),
    ("synthetic env step + next-obs normalise", "env_step",
     hbm(N * (D + A) * 4 + N * 3 * D * 4 + N * 6), 3),
    ("n-step emit counts + scan", "nstep_count", hbm(N * 8), 4),
    ("n-step assemble + ring insert", "nstep_emit", hbm(N * 5414), 5),
    ("state-buffer insert", "state_insert", hbm(2 * N * D * 4), 7),
]


def rows(path):
    r = list(csv.reader(open(path)))
    hdr, units, vals = r[0], r[1], r[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    out = []
    for v in vals:
        def num(key, scale=None):
            if key not in ix or v[ix[key]] in ("", "n/a"):
                return None
            x = float(v[ix[key]].replace(",", ""))
            u = units[ix[key]]
            mult = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                    "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                    "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
            return x * mult
        out.append(dict(name=v[ix["Kernel Name"]], grid=v[ix["Grid Size"]],
                        t=num("gpu__time_duration.sum"),
                        dram=(num("dram__bytes_read.sum") or 0) + (num("dram__bytes_write.sum") or 0),
                        tc=num("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed")))
    return out


def table(title, spec, data, offset=0, positional=False):
    print(f"\n### {title}\n")
    print("| kernel | grid | ncu us | work | achieved | of binding roof | DRAM traffic | tensor pipe |")
    print("|---|---|---|---|---|---|---|---|")
    tot_t = 0.0
    for k, item in enumerate(spec):
        label, key, w = item[:3]
        bound, work = w[0], w[1]
        r = data[item[3]] if positional else data[offset + k]
        assert key in r["name"], (label, key, r["name"])
        t = r["t"]
        tot_t += t
        if bound == "tensor":
            ach = work / t
            t_mma, t_mem = work / TF32_PEAK, w[2] / HBM_PEAK
            roof = (f"{t_mma / t:.2f} (TF32)" if t_mma >= t_mem
                    else f"{t_mem / t:.2f} (HBM, {w[2] / 1e6:.0f} MB operands)")
            cell = f"{work / 1e9:.2f} GFLOP", f"{ach / 1e12:.0f} TF/s", roof
        else:
            ach = work / t
            cell = f"{work / 1e6:.1f} MB", f"{ach / 1e9:.0f} GB/s", f"{ach / HBM_PEAK:.2f} (HBM)"
        tc = f"{r['tc']:.0f}%" if r["tc"] else "-"
        print(f"| {label} | {r['grid']} | {t * 1e6:.1f} | {cell[0]} | {cell[1]} | {cell[2]} | "
              f"{r['dram'] / 1e6:.1f} MB | {tc} |")
    print(f"\nsum of ncu kernel times: {tot_t * 1e6:.0f} us (cold, serialised)")


def main():
    global HBM_PEAK
    root = Path(__file__).resolve().parents[1]
    if len(sys.argv) > 1:
        d, pat = Path(sys.argv[1]), "all_{}_raw.csv"
    else:
        d, pat = root / "profiles", "r1_ncu_{}.csv"
    try:
        HBM_PEAK = json.loads((root / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] * 1e9
    except (OSError, KeyError, ValueError):
        HBM_PEAK = 6.5e12
    print("# Per-kernel rooflines (B200, config 3)\n")
    print(f"Peaks: TF32 {TF32_PEAK / 1e12:.0f} TFLOP/s (cuBLAS 8192^3, measured), "
          f"HBM {HBM_PEAK / 1e9:.0f} GB/s (MEASURED_PEAKS.json copy bandwidth). "
          "Durations from `ncu --set full --clock-control none` (cold caches, one kernel at a "
          "time), so fractions are conservative; in the CUDA graph with PDL and warm L2 the "
          "update runs faster (bench.py).")
    table("Critic update (CriticLearnerCore::update, B=8192)", CRITIC, rows(d / pat.format("critic")))
    table("Policy update (PolicyLearnerCore::update, B=8192)", POLICY,
          rows(d / pat.format("policy")), offset=1)
    table("Actor step + ingest (16384 envs)", ACTOR, rows(d / pat.format("actor")),
          positional=True)


if __name__ == "__main__":
    main()
