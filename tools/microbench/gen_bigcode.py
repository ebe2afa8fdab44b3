"""Generate bigcode1.inc / bigcode2.inc for peaks.cu's k_bigcode (straight-line code far larger than the
instruction cache: BIG_N FMAs with distinct immediates, 8 accumulators).  Generated at build time
(tools/microbench/run_all.sh), not committed.  usage: python gen_bigcode.py [N]"""
import sys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
with open("bigcode1.inc", "w") as f1, open("bigcode2.inc", "w") as f2:
    for i in range(N):
        imm = 0x3C9E0652 + 0x3D1 * i  # distinct fp32 immediates in [0.0193, 0.024)
        f1.write(f'asm volatile("fma.rn.f32 %0, %1, 0f{imm:08X}, %0;" : "+f"(f[{i % 8}]) : "f"(xf));\n')
        f2.write(f'asm volatile("{{.reg .b64 w; mov.b64 w, 0x{imm:08X}{imm:08X}; fma.rn.f32x2 %0, w, %1, %0;}}" '
                 f': "+l"(a[{i % 8}]) : "l"(x));\n')
