"""Static SASS summary of the hot kernels in libtsb.so (opcode mix, registers,
spills): proves what the sm_100a code issues (TEX for the atlas, no tensor
pipe, LDGSTS/TMA absent by design) and is committed as profiles/<tag>_sass.md.

    python scripts/sass_summary.py r02 > profiles/r02_sass.md
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2506_13348_b200" / "libtsb.so"
KERNELS = [
    ("k_raster_fwd<16, HW>", "_ZN3tsb12k_raster_fwdILi16ELi0EEEvNS_12RasterParamsE"),
    ("k_raster_bwd<atomic>", "_ZN3tsb12k_raster_bwdILb0EEEvNS_15RasterBwdParamsE"),
    ("k_preprocess", "_ZN3tsb12k_preprocessENS_10PrepParamsE"),
    ("k_onesweep<8>", "_ZN3tsb10k_onesweepILi8EEEvNS_12OnesweepArgsE"),
    ("k_dup_tx", "_ZN3tsb8k_dup_txENS_7DupArgsE"),
    ("k_shade", "_ZN3tsb7k_shadeENS_11ShadeParamsE"),
]
FAMILIES = [
    ("tex (TEX/TLD/TLD4)", r"^(TEX|TLD|TLD4|TXQ)\b"),
    ("fp32 FMA/ADD/MUL", r"^(FFMA|FADD|FMUL|FMNMX|FSETP|FSEL|FCHK)\b"),
    ("fp64 (DFMA/DADD/DMUL/DSETP)", r"^(DFMA|DADD|DMUL|DSETP|DMNMX)\b"),
    ("SFU (MUFU)", r"^MUFU\b"),
    ("int/logic", r"^(IMAD|IADD3|IADD|LOP3|SHF|ISETP|LEA|IMNMX|SEL|PRMT|POPC|FLO|BREV|IABS|VIADD|VIMNMX|UIADD3|UIMAD|ULOP3|USHF|UISETP|ULEA|USEL|UMOV|MOV|S2R|S2UR|CS2R|R2UR|LDC|LDCU|ULDC|F2I|I2F|F2F|FRND|I2FP|F2IP)\b"),
    ("shared LDS/STS", r"^(LDS|STS|LDSM|ATOMS)\b"),
    ("global LDG/STG", r"^(LDG|STG)\b"),
    ("local LDL/STL (spills)", r"^(LDL|STL)\b"),
    ("global atomics (RED/ATOMG)", r"^(RED|REDG|ATOMG|ATOM)\b"),
    ("warp (SHFL/VOTE/MATCH/REDUX)", r"^(SHFL|VOTE|VOTEU|MATCH|REDUX|WARPSYNC)\b"),
    ("async copy (LDGSTS/UTMALDG/UBLKCP)", r"^(LDGSTS|UTMALDG|UTMASTG|UBLKCP|UTMACCTL)\b"),
    ("tensor (UTCMMA/HMMA)", r"^(UTCMMA|UTCHMMA|UTCQMMA|HMMA|IMMA)\b"),
    ("control (BRA/BAR/BSSY/...)", r"^(BRA|BAR|BSSY|BSYNC|EXIT|RET|CALL|YIELD|NOP|BREAK|JMP|BMOV|NANOSLEEP|MEMBAR|ERRBAR|CCTL|DEPBAR|WARPGROUP)\b"),
]


def sass(fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, str(LIB)], capture_output=True,
                         text=True).stdout
    ops = []
    for line in out.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            ops.append(m.group(2).split(".")[0])
    return ops


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    res = subprocess.run(["cuobjdump", "-res-usage", str(LIB)], capture_output=True,
                         text=True).stdout
    print(f"# {tag}: static SASS of the hot kernels (`scripts/sass_summary.py`, sm_100a)\n")
    print("Instruction counts are STATIC (per kernel body, not executed); the ncu")
    print("summaries carry the executed counts. Registers/stack from `cuobjdump -res-usage`.\n")
    for label, fn in KERNELS:
        ops = sass(fn)
        if not ops:
            continue
        usage = ""
        for i, l in enumerate(res.splitlines()):
            if fn in l:
                nxt = res.splitlines()[i + 1] if i + 1 < len(res.splitlines()) else ""
                usage = " ".join(re.findall(r"(REG:\d+|STACK:\d+|SHARED:\d+)", nxt))
        cnt = collections.Counter()
        other = collections.Counter()
        for op in ops:
            for name, pat in FAMILIES:
                if re.match(pat, op):
                    cnt[name] += 1
                    break
            else:
                other[op] += 1
        print(f"## `{label}` — {len(ops)} SASS instructions; {usage}\n")
        print("| family | count |\n|---|---:|")
        for name, _ in FAMILIES:
            print(f"| {name} | {cnt[name]} |")
        if other:
            print(f"| other ({', '.join(f'{k} {v}' for k, v in other.most_common(6))}) | "
                  f"{sum(other.values())} |")
        print()


if __name__ == "__main__":
    main()
