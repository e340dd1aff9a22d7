"""SASS evidence for the production kernels (run here, no GPU): `cuobjdump -sass` of libtsm2x.so,
per kernel the counts of the instructions that prove the sm_100a datapath — TMA (UTMALDG /
UBLKCP), mbarriers (SYNCS), FP64 tensor-core MMA (DMMA), tcgen05 MMA (UTCHMMA / UTCMMA), TMEM
loads/stores (LDTM / STTM), packed FP32 (FFMA2), fp64 reductions (REDG.E.ADD.F64), spills (LDL/STL) —
plus the first lines around each key instruction, and ptxas's register / stack / spill line. LDL/STL
in the TMA kernels are the producer lane's pending-copy arrays (the 40-byte stack frame), not
spills. Writes profiles/sass_<tag>.txt.

  python tools/sass_excerpt.py [tag]
"""

import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2002_03258_b200", "libtsm2x.so")

# production kernels (tsm2x.cu dispatch): fp64 8/16-column DMMA passes on the swizzled layout (the
# headline), the fp32 16-column tcgen05 kernel, fp32 FFMA2, TSM2L LDG fallback, prep / finalize
PRODUCTION = [
    ("tsm2r_stream_tma<double, 8, DmmaConsumer<8, 8, true, 65536, true>>  (fp64 n=8 headline, split row blocks)",
     r"tsm2r_stream_tmaIdLi8ENS_12DmmaConsumerILi8ELi8ELb1ELi65536ELb1E"),
    ("tsm2r_stream_tma<double, 16, DmmaConsumer<16, 8, false, 65536, true>>  (fp64 TSM2L single-chunk)",
     r"tsm2r_stream_tmaIdLi16ENS_12DmmaConsumerILi16ELi8ELb0ELi65536ELb1E"),
    ("tsm2r_stream_tma<double, 16, DmmaConsumer<16, 8, true, 65536, true>>  (fp64 n=16)",
     r"tsm2r_stream_tmaIdLi16ENS_12DmmaConsumerILi16ELi8ELb1ELi65536ELb1E"),
    ("tsm2r_stream_tc32<false>  (fp32 n=16, split row blocks, tcgen05 kind::tf32)", r"tsm2r_stream_tc32ILb0E"),
    ("tsm2r_stream_tc32<true>  (fp32 n=16, single-chunk row blocks)", r"tsm2r_stream_tc32ILb1E"),
    ("tsm2r_stream_tma<float, 8, Ffma2Consumer<8>>  (fp32 8-column passes)", r"tsm2r_stream_tmaIfLi8ENS_13Ffma2ConsumerILi8E"),
    ("prep_dyn<double, 8, true, double>", r"prep_dynIdLi8ELb1EdE"),
    ("tsm2_finalize<float>", r"tsm2_finalizeIfE"),
]
KEYS = ["UTMALDG", "UBLKCP", "SYNCS", "DMMA", "UTCHMMA", "UTCMMA", "UTCBAR", "LDTM", "STTM", "FFMA2", "DFMA",
        "REDG", "LDL", "STL", "LDS", "ELECT", "ACQBULK"]


def ptxas_info(symbol):
    """Registers / stack / spill line of `nvcc -Xptxas -v` for the symbol (csrc/build.log)."""
    try:
        log = open(os.path.join(ROOT, "paper_2002_03258_b200", "csrc", "build.log")).read().split("\n")
    except OSError:
        return "(no build.log)"
    for i, l in enumerate(log):
        if "Function properties for " + symbol in l:
            regs = next((x for x in log[i + 1:i + 4] if "Used" in x), "")
            return (log[i + 1].strip() + "; " + regs.replace("ptxas info    :", "").strip())[:200]
    return "(not in build.log)"


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    out = [f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)} (sm_100a) — instruction counts and excerpts of the "
           "production kernels (tools/sass_excerpt.py)\n"]
    for label, pat in PRODUCTION:
        body = next((f for f in funcs if re.match(r"_ZN5tsm2x\d*" + pat, f.split("\n", 1)[0])
                     or re.search(pat, f.split("\n", 1)[0])), None)
        if body is None:
            out.append(f"## {label}\n  (not found)\n")
            continue
        name = body.split("\n", 1)[0].strip()
        lines = [l for l in body.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
        ops = collections.Counter()
        for l in lines:
            m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", l)
            if m:
                ops[m.group(1)] += 1
        counts = {k: sum(v for op, v in ops.items() if op.startswith(k)) for k in KEYS}
        out.append(f"## {label}\n   symbol: {name}\n   instructions: {len(lines)}")
        out.append("   ptxas: " + ptxas_info(name))
        out.append("   " + ", ".join(f"{k}={v}" for k, v in counts.items() if v))
        shown = set()
        for key in ("UTMALDG", "UBLKCP", "DMMA", "UTCHMMA", "UTCMMA", "LDTM", "STTM", "FFMA2", "REDG", "SYNCS"):
            for i, l in enumerate(lines):
                if re.search(r"\*/\s+(?:@!?U?P\w+\s+)?" + key, l) and key not in shown:
                    shown.add(key)
                    out.append(f"   -- first {key}:")
                    for x in lines[max(0, i - 1):i + 2]:
                        out.append("     " + re.sub(r"\s+", " ", x.strip())[:150])
                    break
        out.append("")
    path = os.path.join(ROOT, "profiles", f"sass_{tag}.txt")
    with open(path, "w") as fh:
        fh.write("\n".join(out))
    print("\n".join(out)[:6000])


if __name__ == "__main__":
    main()
