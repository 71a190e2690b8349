"""Host emulation of the NVRTC tile passes of one program (debug tool, CPU only).

A GPU run with HHLSV_JIT_DUMP=DIR HHLSV_EMU_DUMP=DIR writes every pass's CUDA source
(tile_<hash>.cu), the program's blob (blob.bin) and the launch list (program.txt). This script
compiles each pass source as host C++ (one std::thread per CUDA thread, std::barrier for
__syncthreads, memcpy for cp.async) and runs the launch list on a state, so a wrong pass can be
found without a GPU-side sanitizer.

    python scripts/jit_emulate.py DIR psi0.npy out.npy
"""
import os
import re
import subprocess
import sys

import numpy as np

SHIM = r'''
#include <cmath>
#include <cstring>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <barrier>
#include <vector>
struct double2 { double x, y; };
struct dim3s { unsigned x, y, z; };
static thread_local dim3s threadIdx;
static dim3s blockIdx, gridDim;
static std::barrier<> *g_bar;
static inline void __syncthreads() { g_bar->arrive_and_wait(); }
template <class T> static inline T __ldg(const T *p) { return *p; }
#define __device__
#define __forceinline__ inline
#define __global__
#define __restrict__
#define __launch_bounds__(a, b)
#define __align__(x)
static unsigned char *g_smem;
#define smem_raw g_smem
static inline unsigned long long __cvta_generic_to_shared(void *p) { return (unsigned long long)p; }
static inline double __ddiv_rn(double a, double b) { return a / b; }
template <class T> static inline T __ldcs(const T *p) { return *p; }
template <class T> static inline void __stcs(T *p, T v) { *p = v; }
'''

MAIN = r'''
int main(int argc, char **argv) {
    const char *psi_path = argv[1], *blob_path = argv[2];
    const unsigned long long n_tiles = strtoull(argv[3], 0, 10), rank_base = strtoull(argv[4], 0, 10);
    const unsigned NTHR = (unsigned)atoi(argv[5]);
    g_smem = (unsigned char *)aligned_alloc(16, (size_t)atoll(argv[6]));   // exact size: ASan sees overruns
    FILE *f = fopen(psi_path, "rb"); fseek(f, 0, SEEK_END); size_t N = ftell(f) / 16; fseek(f, 0, SEEK_SET);
    std::vector<double2> psi(N); fread(psi.data(), 16, N, f); fclose(f);
    f = fopen(blob_path, "rb"); fseek(f, 0, SEEK_END); size_t B = ftell(f) / 16; fseek(f, 0, SEEK_SET);
    std::vector<double2> blob(B); fread(blob.data(), 16, B, f); fclose(f);
    gridDim.x = (unsigned)n_tiles;
    for (unsigned long long t = 0; t < n_tiles; t++) {
        blockIdx.x = (unsigned)t;
        std::barrier<> bar(NTHR); g_bar = &bar;
        std::vector<std::thread> th;
        for (unsigned i = 0; i < NTHR; i++)
            th.emplace_back([&, i] { threadIdx.x = i; threadIdx.y = threadIdx.z = 0;
                                     hhlsv_tile(psi.data(), blob.data(), n_tiles, rank_base); });
        for (auto &x : th) x.join();
    }
    f = fopen(psi_path, "wb"); fwrite(psi.data(), 16, N, f); fclose(f);
}
'''


def host_source(src: str) -> str:
    s = src.replace('extern "C" __global__', "static")
    s = s.replace("extern __shared__ __align__(16) unsigned char smem_raw[];", "")
    s = re.sub(r"__device__ __forceinline__ void cp_async16\(void \*smem, const void \*gmem\) \{.*?\n\}",
               "__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) { memcpy(smem, gmem, 16); }",
               s, flags=re.S)
    s = re.sub(r"void cp_async_(commit|wait1|wait0)\(\) \{[^}]*\}", r"void cp_async_\1() {}", s)
    s = s.replace("#pragma unroll 1", "")
    # prelude: explicit shared-window asm accessors -> byte offsets into the emulated smem
    s = s.replace("__cvta_generic_to_shared(smem_raw)", "0")
    acc = {
        "double2 lds(u32 a)": "{ double2 v; memcpy(&v, g_smem + a, 16); return v; }",
        "void sts(u32 a, double2 v)": "{ memcpy(g_smem + a, &v, 16); }",
        "u64 lds64(u32 a)": "{ u64 v; memcpy(&v, g_smem + a, 8); return v; }",
        "void sts64(u32 a, u64 v)": "{ memcpy(g_smem + a, &v, 8); }",
        "void stsd(u32 a, double v)": "{ memcpy(g_smem + a, &v, 8); }",
        "void bar()": "{ __syncthreads(); }",
        "void cp_async16s(u32 s, const void *gmem)": "{ memcpy(g_smem + s, gmem, 16); }",
    }
    for sig, body in acc.items():
        s = re.sub(r"(__device__ __forceinline__ " + re.escape(sig) + r") \{.*?\n?\}\n", lambda m: m.group(1) + " " + body + "\n",
                   s, count=1, flags=re.S)
    s = re.sub(r'asm volatile\("prefetch\.global\.L2 \[%0\];" ::"l"\(.*?\)\);', ";", s)
    main = MAIN
    if "struct CWArg" in s:
        main = main.replace("hhlsv_tile(psi.data(), blob.data(), n_tiles, rank_base);",
                            "hhlsv_tile(psi.data(), blob.data(), n_tiles, rank_base, g_cw);")
        main = main.replace("int main(int argc, char **argv) {",
                            "static CWArg g_cw;\nint main(int argc, char **argv) {\n    { FILE *c = fopen(argv[7], \"rb\"); "
                            "fread(&g_cw, 1, sizeof g_cw, c); fclose(c); }")
    return SHIM + s + main


def main():
    d, psi0, out = sys.argv[1], sys.argv[2], sys.argv[3]
    psi = np.load(psi0).astype(np.complex128)
    work = os.path.join(d, "emu")
    os.makedirs(work, exist_ok=True)
    state = os.path.join(work, "psi.bin")
    psi.tofile(state)
    for ln in open(os.path.join(d, "program.txt")):
        t = ln.split()
        if t[0] != "TILE":
            raise SystemExit(f"non-tile step in the program: {ln.strip()}")
        tag, n_tiles, T, rb, smem = t[1], int(t[2]), int(t[3]), int(t[4]), int(t[5])
        cwf = os.path.join(d, f"cw_{t[6]}.bin") if len(t) > 6 else "/dev/null"
        exe = os.path.join(work, tag)
        if not os.path.exists(exe):
            src = open(os.path.join(d, tag + ".cu")).read()
            cpp = exe + ".cpp"
            open(cpp, "w").write(host_source(src))
            subprocess.run(["g++", "-O1", "-g", "-std=c++20", "-pthread", "-w", "-fsanitize=address", "-o", exe, cpp],
                           check=True)
        subprocess.run([exe, state, os.path.join(d, "blob.bin"), str(n_tiles), str(rb), str(1 << (T - 4)),
                        str(smem), cwf], check=True)
        print(f"ran {tag} n_tiles={n_tiles}", flush=True)
    np.save(out, np.fromfile(state, dtype=np.complex128))


if __name__ == "__main__":
    main()
