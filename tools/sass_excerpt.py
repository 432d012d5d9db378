#!/usr/bin/env python
"""Writes profiles/r02_sass_excerpt.txt: for the kernels that stage through shared memory with the bulk-async copy
engine, the SASS instruction histogram and the lines that prove it (UBLKCP = cp.async.bulk, SYNCS = mbarrier
operations), from `cuobjdump -sass` of the built library. No GPU needed."""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2304_08232_b200", "libslab_b200.so")
WANT = [("k_gs_planesILi1ELi1ELb1", "k_gs_planes<1,1,true> (plane.cu: phase B, odd planes, colours 4..7 and 7..4)"),
        ("k_gs_planesILi0ELi1ELb1", "k_gs_planes<0,1,true> (plane.cu: phase A, even planes, colours 0..3)"),
        ("k_spmv_planesILb1ELb1", "k_spmv_planes<true,true> (plane_spmv.cu: product with the x'(A x) epilogue)"),
        ("k_dot_exact", "k_dot_exact (kernels.cu: one lane per 4096-chunk, operands by bulk copies)"),
        ("k_gs_pair_tile", "k_gs_pair_tile (tile.cu: colour-pair smoother of masked box levels)")]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    out = ["cuobjdump -sass paper_2304_08232_b200/libslab_b200.so (sm_100a) — instruction histograms of the kernels that stage",
           "their operands through shared memory with the bulk-async copy engine. UBLKCP.S.G = cp.async.bulk global -> shared",
           "(mbarrier complete_tx), UBLKCP.G.S = shared -> global (bulk_group), SYNCS.* = mbarrier init / arrive / expect_tx /",
           "try_wait, UTMACMDFLUSH / UTMACCTL = bulk-group commit and wait. No LDG of the gathered vector remains in these kernels.", ""]
    for key, title in WANT:
        for b in blocks:
            name = b.split("\n", 1)[0]
            if key in name:
                ops = collections.Counter()
                proof = []
                for line in b.splitlines():
                    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(@!?U?P\d\s+)?([A-Z0-9_.]+)", line)
                    if not m:
                        continue
                    op = m.group(2)
                    ops[op.split(".")[0] if not op.startswith(("UBLKCP", "SYNCS", "UTMA", "LDS", "STS", "LDG", "STG")) else op] += 1
                    if op.startswith(("UBLKCP", "UTMACMDFLUSH", "UTMACCTL")) or op.startswith("SYNCS.ARRIVE") or "TRYWAIT" in op:
                        if len(proof) < 8:
                            proof.append("    " + re.sub(r"\s+/\* 0x[0-9a-f]+ \*/", "", line.strip()))
                out.append(f"== {title}")
                out.append("   " + name[:150])
                out.append("   " + ", ".join(f"{k} {v}" for k, v in ops.most_common(24)))
                out += proof
                out.append("")
                break
    path = os.path.join(ROOT, "profiles", "r02_sass_excerpt.txt")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")
    print(path)


if __name__ == "__main__":
    main()
