"""Instruction-class evidence from the built sm_100a code (cuobjdump -sass libvalve.so): per hot
kernel, the counts of the SASS mnemonics that prove what it runs on -- tcgen05 MMAs (UTCHMMA),
TMA loads (UTMALDG) / bulk copies (UBLKCP), TMEM loads (LDTM), mbarrier ops (SYNCS), the copy's
128-bit global loads / stores, the decision kernel's warp reductions (CREDUX / REDUX), shared
atomics and barriers.  usage: python tools/sass_summary.py [lib] > profiles/r2_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = {
    "k_offline_gemm_pair": ["UTCHMMA", "UTMALDG", "UTCBAR", "LDTM", "SYNCS", "STG"],
    "k_offline_gemm": ["UTCHMMA", "UTMALDG", "UTCBAR", "LDTM", "SYNCS", "STG"],
    "k_reclaim_copy_tma": ["UBLKCP", "SYNCS", "LDG", "STG"],
    "k_reclaim_copy": ["LDG", "STG", "BAR"],
    "k_offline_decode": ["LDG", "FFMA", "ATOMG", "YIELD"],
    "k_reclaim_rows": ["MATCH", "SHFL", "LDG", "STG"],
    "k_reclaim_fused": ["CREDUX", "MATCH", "REDUX", "ATOMS", "BAR", "SHFL", "LDS", "STS"],
    "k_restore_scatter": ["LDG", "STG"],
}


def main(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    print(f"# cuobjdump -sass {os.path.relpath(lib, ROOT)} (sm_100a); mnemonic counts per kernel, width suffixes kept")
    for chunk in re.split(r"\n\s+Function : ", sass)[1:]:
        name = chunk.split("\n", 1)[0].strip()
        short = next((k for k in KERNELS if re.search(r"\d" + k + r"E", name)), None)
        if short is None:
            continue
        counts = collections.Counter()
        for m in re.finditer(r"\b(" + "|".join(KERNELS[short]) + r")((?:\.[A-Z0-9_]+)*)", chunk):
            counts[m.group(1) + m.group(2)] += 1
        n_instr = len(re.findall(r"/\*[0-9a-f]{4}\*/", chunk))
        print(f"{short:22s} instrs={n_instr:5d}  " + "  ".join(f"{k}={v}" for k, v in sorted(counts.items())))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2604_07874_b200", "libvalve.so"))
