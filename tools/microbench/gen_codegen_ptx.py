"""PTX version of the codegen probe (see gen_codegen_probe.py): explicit registers, the X load of
column c+1 issued before the FMAs of column c, weights as immediates.  Lets us time ptxas on
nnz-sized straight-line code and measure instruction-fetch cost on the B200.

usage: python gen_codegen_ptx.py U P out.ptx
"""
import random
import struct
import sys

R, V = 64, 2
U = int(sys.argv[1])
P = int(sys.argv[2])
DENS = 0.1
XCOLS = 256

rng = random.Random(0)
L = []
L.append(".version 8.8\n.target sm_100a\n.address_size 64\n")
L.append(".extern .shared .align 16 .b8 xs[];")
L.append(".visible .entry probe(.param .u64 out, .param .u32 iters, .param .u64 clk, .param .u32 nvar)")
L.append(".maxntid 128, 1, 1\n.minnctapersm 1\n{")
L.append("  .reg .pred %p<8>; .reg .b32 %r<32>; .reg .b64 %rd<16>; .reg .f32 %a<" + str(R * V) + ">; .reg .f32 %x<4>; .reg .f32 %s;")
L.append("  mov.u32 %r0, %tid.x; and.b32 %r1, %r0, 31; shr.u32 %r2, %r0, 5;")
L.append("  ld.param.u32 %r3, [nvar]; rem.u32 %r4, %r2, %r3;")  # var
L.append("  ld.param.u32 %r5, [iters];")
# init smem
L.append("  mov.u32 %r6, %r0;")
L.append("INIT: setp.ge.u32 %p0, %r6, " + str(XCOLS * 64) + "; @%p0 bra INITD;")
L.append("  cvt.rn.f32.u32 %s, %r6; mul.f32 %s, %s, 0f3A83126F; shl.b32 %r7, %r6, 2; mov.u32 %r8, xs; add.u32 %r7, %r7, %r8; st.shared.f32 [%r7], %s;")
L.append("  add.u32 %r6, %r6, 128; bra INIT;")
L.append("INITD: bar.sync 0;")
for i in range(R * V):
    L.append("  mov.f32 %%a%d, 0f00000000;" % i)
L.append("  mov.u32 %r9, xs; shl.b32 %r10, %r1, 3; add.u32 %r11, %r9, %r10;")  # lane base: xs + lane*8
L.append("  mov.u64 %rd0, %clock64;")
L.append("  mov.u32 %r12, 0;")
L.append("LOOP: setp.ge.u32 %p1, %r12, %r5; @%p1 bra DONE;")
nfma = 0
for p in range(P):
    L.append("  setp.eq.u32 %%p2, %%r4, %d; @!%%p2 bra V%d;" % (p, p + 1))
    cols = []
    for c in range(U):
        rows = [r for r in range(R) if rng.random() < DENS]
        if rows:
            cols.append((c, rows))
    # software pipeline: x regs double-buffered (%x0,%x1) / (%x2,%x3)
    def ld(i):
        c = cols[i][0] % XCOLS
        b = 2 * (i & 1)
        return "  ld.shared.v2.f32 {%%x%d, %%x%d}, [%%r11+%d];" % (b, b + 1, c * 256)
    L.append(ld(0))
    for i, (c, rows) in enumerate(cols):
        if i + 1 < len(cols):
            L.append(ld(i + 1))
        b = 2 * (i & 1)
        for r in rows:
            w = struct.unpack("<I", struct.pack("<f", rng.gauss(0, 0.05)))[0]
            L.append("  fma.rn.f32 %%a%d, %%x%d, 0f%08X, %%a%d; fma.rn.f32 %%a%d, %%x%d, 0f%08X, %%a%d;"
                     % (2 * r, b, w, 2 * r, 2 * r + 1, b + 1, w, 2 * r + 1))
            if p == 0:
                nfma += 2
    L.append("  bra NEXT;")
    L.append("V%d:" % (p + 1))
L.append("NEXT: add.u32 %r12, %r12, 1; bra LOOP;")
L.append("DONE: mov.u64 %rd1, %clock64; sub.s64 %rd2, %rd1, %rd0;")
L.append("  mov.f32 %s, 0f00000000;")
for i in range(R * V):
    L.append("  add.f32 %%s, %%s, %%a%d;" % i)
L.append("  setp.eq.f32 %p3, %s, 0f46405800; ld.param.u64 %rd3, [out]; @%p3 st.global.f32 [%rd3], %s;")
L.append("  mov.u32 %r14, %ctaid.x; or.b32 %r13, %r0, %r14; setp.eq.u32 %p4, %r13, 0; ld.param.u64 %rd4, [clk]; @%p4 st.global.u64 [%rd4], %rd2;")
L.append("  ret;\n}")
open(sys.argv[3], "w").write("\n".join(L) + "\n")
print("fma per thread per iter (variant 0):", nfma, "cols", len(cols))
