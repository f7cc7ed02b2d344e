"""SASS instruction summary of the built libraries (cuobjdump -sass): per kernel family, the
counts of the Blackwell instructions that prove the tcgen05 / TMEM / TMA path
(UTCHMMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st, UTMALDG/UTMAREDG = TMA tensor load /
reduce, UBLKCP = bulk copy) and the softmax pipe (MUFU.EX2). Usage: python tools/sass_summary.py"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = [os.path.join(ROOT, "paper_2412_05496_b200", "libflexattn_b200.so"),
        os.path.join(ROOT, "tests", "cpp", "libcustom_mods.so")]
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAREDG", "UTMASTG", "UBLKCP", "MUFU.EX2", "MUFU.TANH",
       "SYNCS.ARRIVE", "SYNCS.PHASECHK"]
FAMILIES = [("fwd_sm100", "flex_fwd_sm100_kernel"), ("fwd1t (long rows)", "flex_fwd1t_kernel"),
            ("bwd_sm100 (fused)", "flex_bwd_sm100_kernel"), ("bwd_dq (dQ pass)", "flex_bwd_dq_kernel"),
            ("bwd_preprocess", "bwd_preprocess_kernel"), ("decode_tc (GQA/multi-row)", "decode_tc_kernel"),
            ("decode", "decode_kernel"), ("block_mask", "classify_kernel"), ("page_pool", "pool_"),
            ("fwd_simt", "fwd_simt_kernel"), ("bwd_simt", "bsimt")]


def main():
    for lib in LIBS:
        if not os.path.exists(lib):
            continue
        sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
        fam_counts = collections.defaultdict(collections.Counter)
        kernels = collections.Counter()
        cur = None
        for line in sass.split("\n"):
            m = re.search(r"Function : (\S+)", line)
            if m:
                cur = next((f for f, key in FAMILIES if key in m.group(1)), "other")
                kernels[cur] += 1
                continue
            if cur is None:
                continue
            for op in OPS:
                if re.search(r"\b" + re.escape(op) + r"[\.\s]", line + " "):
                    fam_counts[cur][op] += 1
        print(f"== {os.path.relpath(lib, ROOT)}  (cuobjdump -sass, sm_100a)")
        for f, _ in FAMILIES + [("other", "")]:
            if kernels[f]:
                ops = ", ".join(f"{op} {fam_counts[f][op]}" for op in OPS if fam_counts[f][op])
                print(f"  {f:20s} {kernels[f]:3d} kernels: {ops}")


if __name__ == "__main__":
    sys.exit(main())
