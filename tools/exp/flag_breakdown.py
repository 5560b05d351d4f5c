"""Debug build: which certification test flags each undecided triplet of the
certified compress pass (K1a), counted over 2^20 keys at b = 2, 3, 4.
Builds a patched library into tools/exp/lib_flags.so (not the product)."""
import os, shutil, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
p = os.path.join(R, "paper_2605_21226_b200/csrc/compress_fast.cu")
orig = open(p).read()
s = orig


def rep(a, b):
    global s
    assert a in s, a[:80]
    s = s.replace(a, b, 1)


rep("template <int BD, int BN, int MODE, int DT, bool QJL>\n__global__", """__device__ unsigned long long g_flagcat[8];
extern "C" int oq_debug_flagcat(unsigned long long* h) {
  return (int)cudaMemcpyFromSymbol(h, g_flagcat, sizeof(g_flagcat));
}
extern "C" int oq_debug_flagcat_reset() {
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return (int)cudaMemcpyToSymbol(g_flagcat, z, sizeof(z));
}
template <int BD, int BN, int MODE, int DT, bool QJL>
__global__""")
rep("        okt = l1 > 1e-6f && (pad || a2 > es) && (up || (a0 > es && a1 > es));",
    "        okt = l1 > 1e-6f && (pad || a2 > es) && (up || (a0 > es && a1 > es));\n        int cat = okt ? 0 : 1;")
rep("        const uint32_t sx = cf_bucket(xi, gx, mylut, okt);\n        const uint32_t sy = cf_bucket(eta, gx, mylut, okt);",
    "        const uint32_t sx = cf_bucket(xi, gx, mylut, okt);\n        if (!okt && !cat) cat = 2;\n        const uint32_t sy = cf_bucket(eta, gx, mylut, okt);\n        if (!okt && !cat) cat = 3;")
i = s.index("okt = okt && (b1 - b2 >")
j = s.index(";", i)
s = s[:j + 1] + "\n          if (!okt && !cat) cat = 4;" + s[j + 1:]
rep("        gmask |= (okt ? 0u : 1u) << j;", "        if (!okt && !cat) cat = 5;\n        if (cat) atomicAdd(&g_flagcat[cat], 1ull);\n        gmask |= (okt ? 0u : 1u) << j;")
lib = os.path.join(R, "paper_2605_21226_b200/liboctoquant_b200.so")
try:
    open(p, "w").write(s)
    subprocess.run(["make", "-C", R, "-j16"], check=True, capture_output=True)
    shutil.copy(lib, os.path.join(R, "tools/exp/lib_flags.so"))
finally:
    open(p, "w").write(orig)
    subprocess.run(["make", "-C", R, "-j16"], check=True, capture_output=True)
print("built tools/exp/lib_flags.so")
