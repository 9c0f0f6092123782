"""Per-kernel SASS opcode counts of the built library (evidence that the hot kernels use the
Blackwell paths: UTCHMMA / LDTM / UTCBAR (tcgen05 MMA, TMEM loads, commits), UBLKCP + SYNCS
(cp.async.bulk + mbarrier), FFMA2 / FMUL2 / FADD2 (packed FP32)).

    python tools/sass_evidence.py [lib.so] > profiles/r2_sass_counts.txt
"""
import collections
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "SYNCS", "FFMA2", "FMUL2", "FADD2", "FFMA",
       "MUFU", "SHFL", "LDS", "STS", "LDG", "STG", "RED", "ATOMS"]
KERNELS = ["k_landau_sym", "k_sym_fold", "k_sym_tiles", "k_landau_x2", "k_silu<", "k_silu_finalize",
           "k_blob_sym", "k_push", "k_deposit_bulk_ws", "k_radix_scatter_b", "k_radix_count",
           "k_collision_epilogue", "k_mlp_forward", "k_ism_partials"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_25832_b200/lib/libscorepic_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    dem = subprocess.run(["c++filt"], input="\n".join(f.split("\n")[0].strip() for f in funcs),
                         capture_output=True, text=True).stdout.split("\n")
    print(f"cuobjdump -sass {so}: opcode counts (static instructions) per kernel")
    print("kernel".ljust(72) + "".join(o.rjust(8) for o in OPS))
    for name, body in zip(dem, funcs):
        if not any(k in name for k in KERNELS):
            continue
        ops = collections.Counter()
        for m in re.finditer(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)", body):
            ops[m.group(1)] += 1
        short = re.sub(r"\(.*", "", name.replace("spic::", "").replace("(anonymous namespace)::", ""))
        print(short[:71].ljust(72) + "".join(str(ops.get(o, 0)).rjust(8) for o in OPS))


if __name__ == "__main__":
    main()
