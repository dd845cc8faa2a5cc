"""Per-kernel SASS instruction summary of libchebstep_gpu.so (no GPU needed).

    python tools/sass_summary.py [--lib paper_2603_09790_b200/lib/libchebstep_gpu.so] [--all]

For each hot kernel: instruction count, FP64 tensor-core ops (DMMA), bulk /
tensor copies (UBLKCP = cp.async.bulk, UTMALDG = TMA tensor load), mbarrier
ops (SYNCS), global load/store widths (LDG/STG .64/.128), shared-memory ops,
DFMA/DADD/DMUL, and registers/shared memory from cuobjdump -res-usage.
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOT = ("sell_boxsep_kernel", "update_tr_kernel", "lz2_resid_proj_kernel", "lz2_cgs_kernel",
       "lz2_scale_kernel", "sell_box_kernel", "sell_kernel", "sell_zb_kernel", "update_kernel", "update_gram_kernel",
       "pack_kernel", "fast_step_kernel", "fast_setup_kernel", "proj_kernel", "cgs_kernel",
       "tree_gram_kernel", "resid_kernel", "bj_apply_kernel", "pcg_vec_kernel", "csr_fill_kernel")
KEYS = ("DMMA", "DFMA", "DADD", "DMUL", "UBLKCP", "UTMALDG", "SYNCS", "LDG.E.128", "LDG.E.64",
        "LDG.E.ENL2", "STG.E.128", "STG.E.64", "LDS", "STS", "SHFL", "BAR", "ST.E", "LD.E")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2603_09790_b200", "lib",
                                                  "libchebstep_gpu.so"))
    ap.add_argument("--all", action="store_true")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", a.lib], capture_output=True, text=True).stdout
    usage = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
        if cur and m:
            usage[cur] = (int(m.group(1)), int(m.group(2)))
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if cur and m:
            op = m.group(2)
            c = funcs[cur]
            c["_total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + ".") or (k.endswith(".128") and op.startswith(k)) \
                        or (k in ("LDG.E.64", "STG.E.64") and op.startswith(k)):
                    c[k] += 1
            if op.startswith("LDG"):
                c["LDG*"] += 1
            if op.startswith("STG"):
                c["STG*"] += 1
    names = list(funcs)
    dem = dict(zip(names, demangle(names)))
    rows = []
    for mang, c in funcs.items():
        d = dem[mang]
        if not a.all and not any(h in d for h in HOT):
            continue
        reg, shm = usage.get(mang, (None, None))
        short = d.replace("(anonymous namespace)::", "").replace("void ", "").replace("csg::", "")
        short = re.sub(r"\(.*", "", short)
        rows.append((short, reg, shm, c))
    keys = ["_total", "DMMA", "DFMA", "DADD", "DMUL", "UBLKCP", "UTMALDG", "SYNCS", "LDG*",
            "LDG.E.128", "STG*", "STG.E.128", "LDS", "STS", "SHFL", "BAR"]
    print("kernel | REG | SHARED | " + " | ".join(k.strip("_") for k in keys))
    for short, reg, shm, c in sorted(rows):
        print(f"{short} | {reg} | {shm} | " + " | ".join(str(c.get(k, 0)) for k in keys))


if __name__ == "__main__":
    main()
