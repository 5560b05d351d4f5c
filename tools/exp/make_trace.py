"""Build tools/exp/lib_trace.so: the library with %globaltimer stamps at the
K3 phase boundaries (CTA thread 0) and an oq_debug_trace() export.
Stamps: 0 kernel start, 1 table ready, then per segment (up to 2) qprep done,
tiles done, state out, merge stored, arrival done, segment end."""
import os, shutil, subprocess
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
p = os.path.join(R, "paper_2605_21226_b200/csrc/attention.cu")
orig = open(p).read()
s = orig


def rep(a, b):
    global s
    assert a in s, a[:80]
    s = s.replace(a, b, 1)


rep("extern __shared__ __align__(1024) uint8_t g_attn_smem[];", """extern __shared__ __align__(1024) uint8_t g_attn_smem[];
__device__ unsigned long long g_trace[148][16];
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
#define TR(k) do { if (threadIdx.x == 0 && (k) < 16) g_trace[blockIdx.x][k] = gtime(); } while (0)""")
i = s.index("attn_partials_kernel(const AttnKParams P) {")
j = s.index("\n", i)
s = s[:j + 1] + "  TR(0);\n" + s[j + 1:]
rep("  mbar_wait(&s_tab_bar, 0);\n", "  mbar_wait(&s_tab_bar, 0);\n  TR(1);\n  int segc = 0;\n")
rep("""      load_qfrag(qf, P, it.sh, lane);
    }
""", """      load_qfrag(qf, P, it.sh, lane);
    }
    TR(2 + 6 * segc);
""")
rep("    warp_state_out(S, merge + warp * WS, g, c);", "    TR(3 + 6 * segc);\n    warp_state_out(S, merge + warp * WS, g, c);")
rep("    merge_store<kAttnWarps>(P, it, merge, s_mf, tid, blockDim.x, WS);",
    "    TR(4 + 6 * segc);\n    merge_store<kAttnWarps>(P, it, merge, s_mf, tid, blockDim.x, WS);\n    TR(5 + 6 * segc);")
rep("      __syncthreads();\n      if (s_last && P.p2p_nranks > 0) {", "      __syncthreads();\n      TR(6 + 6 * segc);\n      if (s_last && P.p2p_nranks > 0) {")
rep("""    __syncthreads();
  };

  if (!P.streamk) {""", """    __syncthreads();
    TR(7 + 6 * segc);
    segc = segc < 1 ? segc + 1 : 1;
  };

  if (!P.streamk) {""")
# inside the fused query prep (slots 14, 15: the last segment's values)
rep("""    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) qsw[4 * lane + i] = qkw[4 * lane + i] = 0.f;
    }
  }
  __syncthreads();""", """    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) qsw[4 * lane + i] = qkw[4 * lane + i] = 0.f;
    }
  }
  TR(14);
  __syncthreads();
  TR(15);""")
rep("cudaError_t launch_attention_combine(", """extern "C" int oq_debug_trace(unsigned long long* h) {
  return (int)cudaMemcpyFromSymbol(h, g_trace, sizeof(g_trace));
}

cudaError_t launch_attention_combine(""")
lib = os.path.join(R, "paper_2605_21226_b200/liboctoquant_b200.so")
try:
    open(p, "w").write(s)
    subprocess.run(["make", "-C", R, "-j16"], check=True, capture_output=True)
    shutil.copy(lib, os.path.join(R, "tools/exp/lib_trace.so"))
finally:
    open(p, "w").write(orig)
    subprocess.run(["make", "-C", R, "-j16"], check=True, capture_output=True)
print("built tools/exp/lib_trace.so")
