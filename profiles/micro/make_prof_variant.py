"""Write an instrumented copy of csrc/imgc.cu (clock64 per role and tile,
CTA 0) to /tmp/vsrc/imgc.cu and link alt/prof.so; read with enc_prof.py."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
s = (ROOT / "paper_1203_4938_b200/csrc/imgc.cu").read_text()


def rep(old, new):
    global s
    assert s.count(old) == 1, old[:70]
    s = s.replace(old, new)


s = s.replace("namespace dpp {", """namespace dpp {
__device__ unsigned long long g_prof[2][2][128][8];  // [role][pipeline][tile][event]
#define PROF(role, ev) do { if (blockIdx.x == 0 && lane == 0 && (warp & 3) == 0 && uses < 128) \\
   g_prof[role][b][uses][ev] = clock64(); } while (0)
""", 1)
s = s.replace("""__device__ unsigned long long g_prof[2][2][128][8];  // [role][pipeline][tile][event]
#define PROF(role, ev) do { if (blockIdx.x == 0 && lane == 0 && (warp & 3) == 0 && uses < 128) \\
   g_prof[role][b][uses][ev] = clock64(); } while (0)""", "")
s = s.replace("namespace dpp {", """namespace dpp {
__device__ unsigned long long g_prof[4][64][8];  // [group][group tile][event]
#define PROF(ev) do { if (blockIdx.x == 0 && lane == 0 && (warp & 3) == 0 && gtiles < 64) \\
   g_prof[grp][gtiles][ev] = clock64(); } while (0)
""", 1)
rep("""      // ---------------------------------------------------------------- front
""", """      // ---------------------------------------------------------------- front
      PROF(0);
""")
rep("""      fence_proxy_async_smem();
      ws::named_sync(1 + grp, 128);""", """      PROF(1);
      fence_proxy_async_smem();
      ws::named_sync(1 + grp, 128);
      PROF(2);""")
rep("""        mbar_wait(&tmem_free[slot], (use & 1) ^ 1);
        tc::fence_after();""", """        mbar_wait(&tmem_free[slot], (use & 1) ^ 1);
        PROF(3);
        tc::fence_after();""")
rep("""      mbar_wait(&mma_done[grp], gtiles & 1);
      ++gtiles;""", """      PROF(4);
      mbar_wait(&mma_done[grp], gtiles & 1);
      PROF(5);""")
rep("""      const int i1 = (int)gacc - 1024;""", """      PROF(6);
      const int i1 = (int)gacc - 1024;""")
rep("""    u0 += (uint32_t)nlocal;""", """    u0 += (uint32_t)nlocal;
    (void)0;""")
rep("""          a.idx_plane[gk] = (uint8_t)bj;
        } else {
          uint8_t* rec = a.records + gk * 3;
          rec[0] = mu;
          rec[1] = sg;
          rec[2] = (uint8_t)bj;
        }
      }""", """          a.idx_plane[gk] = (uint8_t)bj;
        } else {
          uint8_t* rec = a.records + gk * 3;
          rec[0] = mu;
          rec[1] = sg;
          rec[2] = (uint8_t)bj;
        }
      }
      PROF(7);
      ++gtiles;""")
s += """
extern "C" int dpp_enc_prof_read(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, dpp::g_prof, sizeof(dpp::g_prof));
}
"""
Path("/tmp/vsrc").mkdir(exist_ok=True)
Path("/tmp/vsrc/imgc.cu").write_text(s)
subprocess.run([sys.executable, str(ROOT / "profiles/micro/build_variant.py"), "prof", "/tmp/vsrc/imgc.cu",
                *sys.argv[1:]], check=True)
