"""Per-kernel counts of the Blackwell-native SASS mnemonics in the built library (cuobjdump, no
GPU needed): UTC*MMA (tcgen05.mma), LDTM / STTM (tcgen05.ld / st), UTMALDG / UBLKCP (TMA / bulk
copies), FFMA2 (packed fp32) -- and the legacy HMMA / HGMMA, which must not appear.

    python scripts/sass_evidence.py [paper_1705_07272_b200/lib/libhaarshift.so] > profiles/sass_evidence.txt
"""
import collections
import os
import re
import subprocess
import sys

MNEMONICS = ("UTCHMMA", "UTCQMMA", "UTCIMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "FFMA2", "HMMA", "HGMMA")


def kernel_counts(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    func = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            func = m.group(1)
            counts.setdefault(func, collections.Counter())
            continue
        if func is None:
            continue
        for mn in MNEMONICS:
            if re.search(r"\b" + mn + r"\b", line):
                counts[func][mn] += 1
    return counts


def short(name):
    """the kernel identifier of an anonymous-namespace mangled name (..._cu_<8 hex><len><name>...)"""
    m = re.search(r"_cu_[0-9a-f]{8}(\d+)", name)
    if m:
        start = m.end()
        ident = name[start:start + int(m.group(1))]
        tmpl = re.search(r"IL(i\d+E)+", name[start + int(m.group(1)):])
        return ident + (("<" + ",".join(re.findall(r"i(\d+)E", tmpl.group(0))) + ">") if tmpl else "")
    return name[:60]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_1705_07272_b200",
                                                             "lib", "libhaarshift.so")
    counts = kernel_counts(lib)
    print(f"# SASS mnemonic counts per kernel of {os.path.basename(lib)} (cuobjdump -sass, sm_100a)")
    for f, c in counts.items():
        if c:
            print(f"{short(f):40s} " + " ".join(f"{k}={v}" for k, v in sorted(c.items())))
    print(f"# {len(counts)} kernels; kernels without any of {', '.join(MNEMONICS)} are omitted")


if __name__ == "__main__":
    main()
