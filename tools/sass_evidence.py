"""SASS evidence that the hot kernels use the Blackwell paths they claim: per kernel, the
tcgen05 / TMEM / bulk-copy / mbarrier instruction counts in the built libarfx.so
(cuobjdump -sass). Usage: python tools/sass_evidence.py [out.md]"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2212_10550_b200" / "lib" / "libarfx.so"
PREFIXES = {
    "UTCHMMA": "tcgen05.mma (kind::f16), issued by one elected thread",
    "UTCBAR": "tcgen05.commit -> mbarrier",
    "UTCATOMSWS": "tcgen05.alloc / dealloc (TMEM columns)",
    "LDTM": "tcgen05.ld (TMEM -> registers, epilogue)",
    "STTM": "tcgen05.st (registers -> TMEM: the next layer's A operand)",
    "UBLKCP": "cp.async.bulk (global -> shared, TMA engine)",
    "SYNCS": "mbarrier arrive / expect-tx / try-wait",
    "ELECT": "elect.sync (single issuing thread)",
    "FENCE.VIEW.ASYNC": "fence.proxy.async (generic -> async proxy)",
}
KERNELS = ["field_fused_kernel", "field_bwd_tc_kernel"]


def main(out=None):
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    lines = ["| kernel | instruction | static count | meaning |", "|---|---|---|---|"]
    for f in re.split(r"\n\s*Function : ", sass)[1:]:
        name = f.split("\n", 1)[0].strip()
        kern = next((k for k in KERNELS if k in name), None)
        if kern is None:
            continue
        ops = collections.Counter(m.group(1) for m in re.finditer(
            r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Za-z0-9_]+)*)", f))
        # template instantiations are told apart by their mangled suffix (e.g. Lb0 / Lb1)
        inst = re.search(r"ILb([01])E", name)
        short = kern + (f"<{'true' if inst.group(1) == '1' else 'false'}>" if inst else "")
        for op, c in sorted(ops.items()):
            for p, meaning in PREFIXES.items():
                if op.startswith(p):
                    lines.append(f"| `{short}` | `{op}` | {c} | {meaning} |")
                    break
    text = "\n".join(lines) + "\n"
    if out:
        Path(out).write_text(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
