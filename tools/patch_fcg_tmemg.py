"""Experiment patch (k_fcgscan.cu): g^ parked in spare TMEM columns (tcgen05.st in phase A,
tcgen05.ld issued before the carry wait in phase C, staged into the quad's dead Bv rows),
freeing the smem G array for a 4th ring stage."""
import re
p = "paper_2406_02528_b200/csrc/k_fcgscan.cu"
s = open(p).read()
def rep(a, b):
    global s
    assert a in s, a[:70]
    s = s.replace(a, b, 1)
rep("constexpr int kFS = 3;                    // ring stages",
    "#ifndef TERN_FS_STAGES\n#define TERN_FS_STAGES 4\n#endif\n"
    "constexpr int kFS = TERN_FS_STAGES;       // ring stages (g^ parked in TMEM makes room for 4)\n"
    "constexpr int kFGCol = 192;               // TMEM columns of g^: the 64 after each accumulator")
rep("  float G[kFBM][kFPad];              // g^\n", "")
rep("""          sm.G[r][cc] = gh0;
          sm.G[r][cc + 1] = gh1;""", """          gq[j] = __float_as_uint(gh0);
          gq[j + 1] = __float_as_uint(gh1);""")
rep("        const int cb = c0 + cs * kFQCh;",
    "        const int cb = c0 + cs * kFQCh;\n"
    "        uint32_t gq[kFQCh];   // g^ of this row's 16 channels -> TMEM until phase C")
rep("""        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ready[quad][half]);   // carry may run these rows""",
"""        // g^ into this warp's own spare TMEM block (its lane quadrant x its 16 columns
        // next to the tile's accumulator): rewritten only by this warp, two tiles later
        const uint32_t gaddr = tmem_base + kFGCol + acc * 256 + cs * kFQCh +
                               ((uint32_t)(quad * 32) << 16);
        if (!a.nogate) tmem_st16(gaddr, gq);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ready[quad][half]);   // carry may run these rows""")
rep("""        const long long w5 = clock64();
        if (a.backoff)""", """        uint32_t gv[kFQCh];   // g^ back from TMEM, its latency hidden behind the carry wait
        if (!a.nogate) {
          tmem_st_wait();
          tmem_ld16(gaddr, gv);
        }
        const long long w5 = clock64();
        if (a.backoff)""")
rep("""        const long long w6 = clock64();
        const int cc = cs * kFQCh + (lane & 15), rsub = lane >> 4;""",
"""        const long long w6 = clock64();
        if (!a.nogate) {   // into the quad's Bv rows: the carry is done with them (hdone)
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < kFQCh; ++j) sm.Bv[r][cs * kFQCh + j] = __uint_as_float(gv[j]);
          __syncwarp();
        }
        const int cc = cs * kFQCh + (lane & 15), rsub = lane >> 4;""")
rep("const float g0 = sm.G[t][cc], g1 = sm.G[t + 1][cc];", "const float g0 = sm.Bv[t][cc], g1 = sm.Bv[t + 1][cc];")
open(p, "w").write(s)
c = "paper_2406_02528_b200/csrc/common.cuh"
s = open(c).read()
if "tmem_st16" not in s:
    a = "__device__ __forceinline__ void tmem_ld_wait() {"
    s = s.replace(a, '''// thread i stores 16 32-bit values to TMEM lane (base+i), cols [col, col+16)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
''' + a, 1)
    open(c, "w").write(s)
print("patched")
