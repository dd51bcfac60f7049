// NVRTC specialisation of pass kernels (host code).
//
// The interpreter kernel (pass_kernel.cu) walks the pass's op records and
// switches over ~40 register-block primitive bodies at run time: ~25 % of its
// instructions are dispatch, the ~200 KB of SASS per variant misses the
// instruction cache (ncu: 11 % `no_inst` stalls) and every CX through a
// rotated slot costs selects.  Here each pass is re-emitted as straight-line
// CUDA source — tile enumeration masks, slot positions, member-rotation table,
// primitive sequence and blob offsets as compile-time constants, matrices still
// read from the SMEM blob — and compiled by NVRTC to sm_100a SASS.  Passes with
// the same structure share one kernel.  Compilation runs in parallel threads
// and the cubins are cached on disk (QSV_JIT_CACHE, default ~/.cache/qsv_jit).
//
// The driver API is reached through cudaGetDriverEntryPoint and NVRTC through
// dlopen, so libqsv.so has no link-time dependency on libcuda or libnvrtc.
#include "qsv_internal.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <thread>
#include <vector>

namespace qsv {

namespace {

const char* kDeviceSource =
#include "jit_src.inc"
    ;

// ------------------------------------------------------------------ loaders
struct Nvrtc {
    bool ok = false;
    std::string why;
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
};

const Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
        void* h = nullptr;
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL)))
                break;
        if (!h) {
            n.why = "libnvrtc.so.12 not found";
            return;
        }
        n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
        n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
        n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
        n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        n.log_size = reinterpret_cast<decltype(n.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
        n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size && n.log && n.destroy;
        if (!n.ok)
            n.why = "libnvrtc is missing symbols";
    });
    return n;
}

struct Driver {
    bool ok = false;
    CUresult (*module_load)(CUmodule*, const void*) = nullptr;
    CUresult (*get_function)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*set_attr)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
    CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                       CUstream, void**, void**) = nullptr;
    CUresult (*unload)(CUmodule) = nullptr;
    CUresult (*encode_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
};

template <typename F>
bool entry(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p)
        return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

const Driver& driver() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = entry("cuModuleLoadData", d.module_load) && entry("cuModuleGetFunction", d.get_function) &&
               entry("cuFuncSetAttribute", d.set_attr) &&
               entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", d.occupancy) &&
               entry("cuLaunchKernel", d.launch) && entry("cuModuleUnload", d.unload);
        if (!entry("cuTensorMapEncodeTiled", d.encode_tiled))
            d.encode_tiled = nullptr;  // tensor-map tile copies off
    });
    return d;
}

// ------------------------------------------------------------------ codegen
int env_int(const char* name, int dflt, int lo, int hi);

// Split register blocks (two threads per 16-member group, 256 threads for 11-qubit
// tiles, 3 CTAs/SM at 80 registers): measured slower than one thread per group
// (random-30 345 vs 310 ms, HEA-30 133 vs 120 ms; profiles/README.md), so opt-in
// with QSV_JIT_SPLIT=1.
bool split_blocks() {
    const char* e = std::getenv("QSV_JIT_SPLIT");
    return e && e[0] == '1';
}
// Wide kernels (set while a kernel is generated, QSV_JIT_WIDE=1): 11-qubit tiles whose
// register blocks hold 8 amplitudes (rblock_k = 3) run 256 threads, one 8-member group each —
// twice the warps per SM at 72-74 registers.  Measured equal to 128 threads (random-30 with
// rblock_k = 3: 381.5 vs 380.5 ms, HEA-30 138.7 vs 136.5), so off by default.
thread_local bool t_wide = false;
int threads_for_k(int K) {
    if (K == 11 && (split_blocks() || t_wide))
        return 256;
    return K >= 12 ? 256 : (K >= 8 ? 128 : (K >= 6 ? 64 : 32));
}

std::string u32(uint32_t x) {
    std::ostringstream o;
    o << "0x" << std::hex << x << "u";
    return o.str();
}

std::string u64(uint64_t x) {
    std::ostringstream o;
    o << "0x" << std::hex << x << "ull";
    return o.str();
}

// Body of one pass (ops applied to one tile) as source text.
// Tile groups per CTA of a specialised pass kernel (pass_pipeline MT).  Default 1: three
// independent CTAs per SM.  QSV_JIT_MT=3 runs 3 lockstep groups of 128 threads per CTA
// (one CTA per SM, all warps on the same code): measured slower — random-30 345 vs 278 ms,
// HEA-30 140 vs 114 ms — because lockstep groups also wait for their loads together,
// which costs more than the instruction-cache misses it saves (profiles/r02_kernel_ab.md).
int jit_mt(int K) {
    const int mt = env_int("QSV_JIT_MT", 1, 1, 3);
    return (K == 11 && !split_blocks()) ? mt : 1;
}

// `mt` > 1: the CTA barrier of an op whose application depends on the tile (out-of-tile
// controls) is hoisted out of the condition so every tile group meets it; ops with
// internal CTA barriers under such a condition make the pass unsuitable (mt_ok = false).
// Class-mode body of a register block (and the diagonal ops / relabel it absorbs): no
// pass-specific constant appears in the text, so passes that differ only in qubit
// positions, tables or blob offsets share one kernel.  Returns the index of the last op
// it consumed.
// (kind, a, b) primitive variants of the program's register blocks (class mode: the rolled
// primitive switch carries exactly these, identical in every kernel of the program)
thread_local const std::vector<int>* t_variants = nullptr;

int gen_rblock_class(std::ostringstream& o, const Step& s, const unsigned char* blob, int i) {
    const int K = s.geom.K;
    const int NT = threads_for_k(K);
    const TileOp* ops = reinterpret_cast<const TileOp*>(blob);
    const TileOp& op = ops[i];
    const int KB = op.k, NV = 1 << KB;
    auto ref = [](int j) {
        return "(*reinterpret_cast<const qsv::TileOp*>(blob + " + std::to_string(j * sizeof(TileOp)) + "))";
    };
    std::ostringstream pre, epib;
    int last = i;
    if (op.xctrl == 0 && op.tctrl == 0 && !std::getenv("QSV_JIT_NO_EPI")) {
        for (int j = i + 1; j < s.nops; ++j) {
            const TileOp& d = ops[j];
            if (d.kind != QSV_OP_DIAG && d.kind != QSV_OP_PHASEPROD && d.kind != QSV_OP_PARPHASE)
                break;
            const std::string J = std::to_string(j), D = "d" + J;
            pre << "  const qsv::TileOp& " << D << " = " << ref(j) << ";\n";
            std::string guard;
            if (d.xctrl) {
                pre << "  const bool on" << J << " = (full_base & " << D << ".xctrl) == " << D << ".xctrl;\n";
                guard = "on" + J;
            }
            if (d.tctrl)
                guard += std::string(guard.empty() ? "" : " && ") + "((idx & " + D + ".tctrl) == " + D + ".tctrl)";
            std::string stmt;
            if (d.kind == QSV_OP_DIAG) {
                pre << "  const double2* g" << J << " = reinterpret_cast<const double2*>(blob + " << D << ".mat_byte);\n"
                    << "  const uint32_t e" << J << " = qsv::diag_ext(" << D << ", full_base);\n";
                if (d.nin == 0) {
                    pre << "  const double2 c" << J << " = g" << J << "[e" << J << "];\n";
                    stmt = "a = qsv::cmul(c" + J + ", a);";
                } else if (d.nin == 1) {
                    pre << "  const double2 c" << J << "a = g" << J << "[e" << J << "], c" << J << "b = g" << J << "[e" << J
                        << " | 1u];\n  const int p" << J << " = __ffs(" << D << ".tmask) - 1;\n";
                    stmt = "a = qsv::cmul(((idx >> p" + J + ") & 1u) ? c" + J + "b : c" + J + "a, a);";
                } else {
                    pre << "  const unsigned char* t" << J << " = blob + " << D << ".ptab_byte;\n";
                    stmt = "a = qsv::cmul(g" + J + "[e" + J + " | t" + J + "[idx & 31u] | t" + J + "[32u + (idx >> 5)]], a);";
                }
            } else if (d.kind == QSV_OP_PHASEPROD) {
                pre << "  const double2* g" << J << " = reinterpret_cast<const double2*>(blob + " << D << ".mat_byte);\n"
                    << "  const double2 c" << J << " = qsv::pp_const(" << D << ", blob, full_base);\n";
                stmt = "a = qsv::cmul(qsv::cmul(c" + J + ", qsv::cmul(g" + J + "[1u + (idx & 31u)], g" + J +
                       "[33u + (idx >> 5)])), a);";
            } else {
                pre << "  double2 c" << J << "a, c" << J << "b;\n  qsv::par_consts(" << D << ", blob, full_base, c" << J
                    << "a, c" << J << "b);\n";
                stmt = "a = qsv::cmul((__popc(idx & " + D + ".tmask) & 1) ? c" + J + "b : c" + J + "a, a);";
            }
            for (int jm = 0; jm < NV; ++jm)
                epib << "    { double2& a = v[" << jm << "]; const uint32_t idx = base ^ (" << ((jm & 1) ? "m0" : "0u")
                     << " | " << ((jm & 2) ? "m1" : "0u") << " | " << ((jm & 4) ? "m2" : "0u") << " | "
                     << ((jm & 8) ? "m3" : "0u") << "); (void)idx; " << (guard.empty() ? "" : "if (" + guard + ") ")
                     << stmt << " }\n";
            last = j;
        }
    }
    const bool fold = last + 1 == s.nops - 1 && ops[last + 1].kind == QSV_OP_RELABEL && op.xctrl == 0 &&
                      op.tctrl == 0 && (1 << (K - __builtin_popcount(op.fmask))) == NT &&
                      env_int("QSV_JIT_FOLD_RELABEL", 1, 0, 1);
    uint32_t rot = 0;
    for (int l = 0; l < 8; ++l)
        rot |= (op.rot_tab >> (4 * l)) & 15u;
    o << pre.str();
    o << "  const qsv::DevPrim* prs" << i << " = reinterpret_cast<const qsv::DevPrim*>(blob + " << ref(i) << ".prim_byte);\n";
    o << "  qsv::jit_rblock_rt<" << K << ", " << NT << ", " << KB << (fold ? ", true" : ", false") << ">(tile, " << ref(i)
      << ", [&](double2 (&v)[" << NV << "], uint32_t& r) {\n    (void)r;\n";
    const DevPrim* pr = reinterpret_cast<const DevPrim*>(blob + op.prim_byte);
    if (env_int("QSV_JIT_CLASS_ROLL", 1, 0, 1)) {
        // rolled: one loop over the block's primitive records, a switch over every
        // (kind, a, b) variant of a KB-qubit block; the rotation is applied at run time
        o << "#pragma unroll 1\n    for (int p = 0; p < " << ref(i) << ".nprim; ++p) {\n"
          << "      const qsv::DevPrim q = prs" << i << "[p];\n"
          << "      const double2* m = reinterpret_cast<const double2*>(blob + q.data_byte); (void)m;\n"
          << "      switch ((q.kind << 4) | (q.a << 2) | q.b) {\n";
        auto want = [&](int key) {
            return !t_variants || std::find(t_variants->begin(), t_variants->end(), key) != t_variants->end();
        };
        for (int a = 0; a < KB; ++a) {
            const char* u1[3] = {"rb_u1", "rb_u1r", "rb_u1i"};
            const int u1k[3] = {QSV_PRIM_U1, QSV_PRIM_U1R, QSV_PRIM_U1I};
            for (int t = 0; t < 3; ++t)
                if (want((u1k[t] << 4) | (a << 2)))
                    o << "      case " << ((u1k[t] << 4) | (a << 2)) << ": qsv::" << u1[t] << "<" << NV << ", " << a
                      << ">(v, m + 4u * ((r >> " << a << ") & 1u)); break;\n";
            for (int b = 0; b < KB; ++b) {
                if (b == a)
                    continue;
                if (want((QSV_PRIM_CX << 4) | (a << 2) | b))
                    o << "      case " << ((QSV_PRIM_CX << 4) | (a << 2) | b) << ": qsv::rb_cx_plain<" << NV << ", "
                      << a << ", " << b << ">(v); r ^= ((r >> " << a << ") & 1u) << " << b << "; break;\n";
                if (b > a && want((QSV_PRIM_U2 << 4) | (a << 2) | b))
                    o << "      case " << ((QSV_PRIM_U2 << 4) | (a << 2) | b) << ": qsv::rb_u2<" << NV << ", " << a
                      << ", " << b << ">(v, m + 16u * (((r >> " << a << ") & 1u) | (((r >> " << b
                      << ") & 1u) << 1))); break;\n";
            }
        }
        if (want((QSV_PRIM_DIAG16 << 4) | (3 << 2) | 3))
            o << "      case " << ((QSV_PRIM_DIAG16 << 4) | (3 << 2) | 3) << ": qsv::rb_diag<" << NV
              << ">(v, m, r); break;\n";
        o << "      default: break;\n      }\n    }\n";
    } else
    for (int p = 0; p < op.nprim; ++p) {
        const DevPrim& q = pr[p];
        const std::string mat = "reinterpret_cast<const double2*>(blob + prs" + std::to_string(i) + "[" +
                                std::to_string(p) + "].data_byte)";
        const bool ra = (rot >> q.a) & 1u, rb = (rot >> q.b) & 1u;
        switch (q.kind) {
        case QSV_PRIM_U1:
        case QSV_PRIM_U1R:
        case QSV_PRIM_U1I: {
            const char* fn = q.kind == QSV_PRIM_U1 ? "rb_u1" : (q.kind == QSV_PRIM_U1R ? "rb_u1r" : "rb_u1i");
            o << "    qsv::" << fn << "<" << NV << ", " << int(q.a) << ">(v, " << mat;
            if (ra)
                o << " + 4u * ((r >> " << int(q.a) << ") & 1u)";
            o << ");\n";
            break;
        }
        case QSV_PRIM_U2:
            o << "    qsv::rb_u2<" << NV << ", " << int(q.a) << ", " << int(q.b) << ">(v, " << mat;
            if (ra || rb)
                o << " + 16u * (((r >> " << int(q.a) << ") & 1u) | (((r >> " << int(q.b) << ") & 1u) << 1))";
            o << ");\n";
            break;
        case QSV_PRIM_CX:
            o << "    qsv::rb_cx_plain<" << NV << ", " << int(q.a) << ", " << int(q.b) << ">(v);\n";
            if (ra) {
                o << "    r ^= ((r >> " << int(q.a) << ") & 1u) << " << int(q.b) << ";\n";
                rot |= 1u << q.b;
            }
            break;
        default:
            o << "    qsv::rb_diag<" << NV << ">(v, " << mat << ", " << (rot ? "r" : "0u") << ");\n";
            break;
        }
    }
    o << "  }, [&](double2 (&v)[" << NV << "], uint32_t base, uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {\n"
      << "    (void)v; (void)base; (void)m0; (void)m1; (void)m2; (void)m3;\n" << epib.str() << "  }";
    if (fold)
        o << ", &" << ref(last + 1);
    o << ");\n";
    return fold ? last + 1 : last;
}

std::string gen_ops(const Step& s, const unsigned char* blob, int& minb, int mt = 1, bool* mt_ok = nullptr,
                    bool class_mode = false) {
    const int K = s.geom.K;
    const int NT = threads_for_k(K);
    const TileOp* ops = reinterpret_cast<const TileOp*>(blob);
    std::ostringstream o;
    minb = K >= 12 ? 1 : 3;
    if (mt_ok)
        *mt_ok = true;
    for (int i = 0; i < s.nops; ++i) {
        const TileOp& op = ops[i];
        const std::string opref = "*reinterpret_cast<const qsv::TileOp*>(blob + " +
                                  std::to_string(i * sizeof(TileOp)) + ")";
        o << "  {\n";
        if (op.xctrl && mt > 1) {
            if (op.kind == QSV_OP_RELABEL || (op.kind == QSV_OP_DENSE && op.k == 5)) {
                if (mt_ok)
                    *mt_ok = false;
            }
            o << "  __syncthreads();\n";
            o << "  if ((full_base & " << u64(op.xctrl) << ") == " << u64(op.xctrl) << ") {\n";
        } else {
            if (op.xctrl && class_mode)
                o << "  if ((full_base & " << opref << ".xctrl) == " << opref << ".xctrl) {\n";
            else if (op.xctrl)
                o << "  if ((full_base & " << u64(op.xctrl) << ") == " << u64(op.xctrl) << ") {\n";
            // the first op's barrier is not needed for correctness (every thread waited on the
            // tile's mbarrier) but keeps the warps in step: without it (QSV_JIT_FIRST_BARRIER=0)
            // random-30 ran 267.1 vs 262.8 ms and UCCSD-24 108.8 vs 105.8 (HEA-30 110.9 vs 113.7)
            if (i > 0 || env_int("QSV_JIT_FIRST_BARRIER", 1, 0, 1))
                o << "  __syncthreads();\n";
        }
        switch (op.kind) {
        case QSV_OP_DENSE:
            if (op.k == 5) {
                o << "  qsv::dense5_op<" << K << ", " << NT << ">(tile, " << opref << ", blob);\n";
                minb = 1;
            } else {
                o << "  qsv::dense_op<" << op.k << ", " << K << ", " << NT << ">(tile, " << opref << ", blob);\n";
            }
            break;
        case QSV_OP_RELABEL:
            o << "  qsv::relabel_op<" << K << ", " << NT << ">(tile, " << opref << ", blob);\n";
            break;
        case QSV_OP_DMMA16:
            o << "  qsv::dmma16_op<" << K << ", " << NT << ">(tile, " << opref << ", blob);\n";
            break;
        case QSV_OP_DIAG:
            o << "  qsv::diag_op<" << K << ", " << NT << ">(tile, " << opref << ", blob, full_base);\n";
            break;
        case QSV_OP_PHASEPROD:
            o << "  qsv::phaseprod_op<" << K << ", " << NT << ">(tile, " << opref << ", blob, full_base);\n";
            break;
        case QSV_OP_PARPHASE:
            o << "  qsv::parphase_op<" << K << ", " << NT << ">(tile, " << opref << ", blob, full_base);\n";
            break;
        case QSV_OP_XPERM:
            o << "  qsv::xperm_op<" << K << ", " << NT << ">(tile, " << opref << ");\n";
            break;
        case QSV_OP_RBLOCK: {
            if (class_mode && !split_blocks()) {
                i = gen_rblock_class(o, s, blob, i);
                break;
            }
            // Diagonal ops right after a whole-tile register block ride along as a
            // per-amplitude epilogue: no extra SMEM sweep or barrier for them.
            std::ostringstream pre, epi, epib;
            int last = i;
            const int KBm = op.k;
            uint32_t mm[4] = {0, 0, 0, 0};
            for (int jj = 0; jj < KBm; ++jj)
                mm[jj] = 1u << op.tpos[jj];
            auto offj = [&](int j) {
                uint32_t o2 = 0;
                for (int bb = 0; bb < KBm; ++bb)
                    if ((j >> bb) & 1)
                        o2 ^= mm[bb];
                return o2;
            };
            const int NVm = 1 << KBm;
            if (op.xctrl == 0 && op.tctrl == 0 && !std::getenv("QSV_JIT_NO_EPI")) {
                for (int j = i + 1; j < s.nops; ++j) {
                    const TileOp& d = ops[j];
                    if (d.kind != QSV_OP_DIAG && d.kind != QSV_OP_PHASEPROD && d.kind != QSV_OP_PARPHASE)
                        break;
                    const std::string dref = "(*reinterpret_cast<const qsv::TileOp*>(blob + " +
                                             std::to_string(j * sizeof(TileOp)) + "))";
                    const std::string J = std::to_string(j);
                    std::string guard;
                    if (d.xctrl) {
                        pre << "  const bool on" << J << " = (full_base & " << u64(d.xctrl) << ") == " << u64(d.xctrl) << ";\n";
                        guard = "on" + J;
                    }
                    if (d.tctrl) {
                        if (!guard.empty())
                            guard += " && ";
                        guard += "((idx & " + u32(d.tctrl) + ") == " + u32(d.tctrl) + ")";
                    }
                    std::string stmt;
                    if (d.kind == QSV_OP_DIAG) {
                        const std::string Dg = "reinterpret_cast<const double2*>(blob + " + std::to_string(d.mat_byte) + ")";
                        pre << "  const uint32_t e" << J << " = qsv::diag_ext(" << dref << ", full_base);\n";
                        if (d.nin == 0) {
                            pre << "  const double2 d" << J << " = " << Dg << "[e" << J << "];\n";
                            stmt = "a = qsv::cmul(d" + J + ", a);";
                        } else if (d.nin == 1) {
                            int pbit = 0;
                            while (!((d.tmask >> pbit) & 1u))
                                ++pbit;
                            pre << "  const double2 d" << J << "a = " << Dg << "[e" << J << "], d" << J << "b = " << Dg
                                << "[e" << J << " | 1u];\n";
                            stmt = "a = qsv::cmul(((idx >> " + std::to_string(pbit) + ") & 1u) ? d" + J + "b : d" + J + "a, a);";
                        } else {
                            const std::string plo = "(blob + " + std::to_string(d.ptab_byte) + ")";
                            stmt = "a = qsv::cmul(" + Dg + "[e" + J + " | " + plo + "[idx & 31u] | " + plo +
                                   "[32u + (idx >> 5)]], a);";
                        }
                    } else if (d.kind == QSV_OP_PHASEPROD) {
                        const std::string tab = "reinterpret_cast<const double2*>(blob + " + std::to_string(d.mat_byte) + ")";
                        pre << "  const double2 c" << J << " = qsv::pp_const(" << dref << ", blob, full_base);\n";
                        stmt = "a = qsv::cmul(qsv::cmul(c" + J + ", qsv::cmul(" + tab + "[1u + (idx & 31u)], " + tab +
                               "[33u + (idx >> 5)])), a);";
                    } else {
                        pre << "  double2 p" << J << "a, p" << J << "b;\n  qsv::par_consts(" << dref
                            << ", blob, full_base, p" << J << "a, p" << J << "b);\n";
                        stmt = "a = qsv::cmul((__popc(idx & " + u32(d.tmask) + ") & 1) ? p" + J + "b : p" + J + "a, a);";
                    }
                    epi << "    " << (guard.empty() ? "" : "if (" + guard + ") ") << stmt << "\n";
                    // block form: per member, with the PHASEPROD table loads shared
                    std::map<uint32_t, std::string> lo_var, hi_var;
                    if (d.kind == QSV_OP_PHASEPROD) {
                        const std::string tab = "reinterpret_cast<const double2*>(blob + " + std::to_string(d.mat_byte) + ")";
                        for (int jm = 0; jm < NVm; ++jm) {
                            const uint32_t lo = offj(jm) & 31u, hi = offj(jm) >> 5;
                            if (!lo_var.count(lo)) {
                                lo_var[lo] = "pa" + J + "_" + std::to_string(lo);
                                epib << "    const double2 " << lo_var[lo] << " = " << tab << "[1u + ((base ^ " << u32(lo)
                                     << ") & 31u)];\n";
                            }
                            if (!hi_var.count(hi)) {
                                hi_var[hi] = "pb" + J + "_" + std::to_string(hi);
                                epib << "    const double2 " << hi_var[hi] << " = " << tab << "[33u + ((base >> 5) ^ " << u32(hi)
                                     << ")];\n";
                            }
                        }
                    }
                    for (int jm = 0; jm < NVm; ++jm) {
                        std::string st = stmt, g = guard;
                        if (d.kind == QSV_OP_PHASEPROD)
                            st = "a = qsv::cmul(qsv::cmul(c" + J + ", qsv::cmul(" + lo_var[offj(jm) & 31u] + ", " +
                                 hi_var[offj(jm) >> 5] + ")), a);";
                        epib << "    { double2& a = v[" << jm << "]; const uint32_t idx = base ^ " << u32(offj(jm))
                             << "; (void)idx; " << (g.empty() ? "" : "if (" + g + ") ") << st << " }\n";
                    }
                    last = j;
                }
            }
            const int KB = op.k;
            const int NV = 1 << KB;
            uint32_t m[4] = {0, 0, 0, 0};
            for (int j = 0; j < KB; ++j)
                m[j] = 1u << op.tpos[j];
            uint32_t rot_any = 0;
            for (int l = 0; l < 8; ++l)
                rot_any |= (op.rot_tab >> (4 * l)) & 15u;
            const DevPrim* prs = reinterpret_cast<const DevPrim*>(blob + op.prim_byte);
            if (KB == 4 && NT == 256 && (1 << (K - __builtin_popcount(op.fmask))) * 2 == NT) {
                // ---- split block: body over 8 registers per thread, re-split on demand
                auto crosses = [&](const DevPrim& q, int S) {
                    switch (q.kind) {
                    case QSV_PRIM_U1: case QSV_PRIM_U1R: case QSV_PRIM_U1I: return q.a == S;
                    case QSV_PRIM_U2: return q.a == S || q.b == S;
                    case QSV_PRIM_CX: return q.b == S;
                    default: return false;
                    }
                };
                auto next_cross = [&](int S, int from) {
                    for (int p = from; p < op.nprim; ++p)
                        if (crosses(prs[p], S))
                            return p;
                    return op.nprim + 1;
                };
                int S = 0;
                for (int c = 1; c < 4; ++c)
                    if (next_cross(c, 0) > next_cross(S, 0))
                        S = c;
                const int S0 = S;
                std::ostringstream body;
                auto loc = [&](int slot) { return slot < S ? slot : slot - 1; };
                for (int p = 0; p < op.nprim; ++p) {
                    const DevPrim& q = prs[p];
                    if (crosses(q, S)) {
                        int best = -1;
                        for (int c = 0; c < 4; ++c) {
                            if (c == S || c == q.a || (q.kind == QSV_PRIM_U2 || q.kind == QSV_PRIM_CX ? c == q.b : false))
                                continue;
                            if (best < 0 || next_cross(c, p) > next_cross(best, p))
                                best = c;
                        }
                        body << "    qsv::rb_resplit<" << S << ", " << best << ">(v, h);\n";
                        S = best;
                    }
                    const std::string mat = "reinterpret_cast<const double2*>(blob + " + std::to_string(q.data_byte) + ")";
                    const bool ra = (rot_any >> q.a) & 1u, rb = (rot_any >> q.b) & 1u;
                    switch (q.kind) {
                    case QSV_PRIM_U1:
                    case QSV_PRIM_U1R:
                    case QSV_PRIM_U1I: {
                        const char* fn = q.kind == QSV_PRIM_U1 ? "rb_u1" : (q.kind == QSV_PRIM_U1R ? "rb_u1r" : "rb_u1i");
                        body << "    qsv::" << fn << "<8, " << loc(q.a) << ">(v, " << mat;
                        if (ra)
                            body << " + 4u * ((r >> " << int(q.a) << ") & 1u)";
                        body << ");\n";
                        break;
                    }
                    case QSV_PRIM_U2:
                        body << "    qsv::rb_u2<8, " << loc(q.a) << ", " << loc(q.b) << ">(v, " << mat;
                        if (ra || rb)
                            body << " + 16u * (((r >> " << int(q.a) << ") & 1u) | (((r >> " << int(q.b) << ") & 1u) << 1))";
                        body << ");\n";
                        break;
                    case QSV_PRIM_CX:
                        if (q.a == S) {
                            body << "    if (h != " << (ra ? "((r >> " + std::to_string(q.a) + ") & 1u)" : std::string("0u"))
                                 << ") qsv::rb_flip<" << loc(q.b) << ">(v);\n";
                        } else if (ra) {
                            body << "    qsv::rb_cx<8, " << loc(q.a) << ", " << loc(q.b) << ">(v, (r & " << ((1 << S) - 1)
                                 << "u) | ((r >> " << (S + 1) << ") << " << S << "));\n";
                        } else {
                            body << "    qsv::rb_cx_plain<8, " << loc(q.a) << ", " << loc(q.b) << ">(v);\n";
                        }
                        break;
                    default:
                        body << "    qsv::rb_diag_split<" << S << ">(v, " << mat << ", " << (rot_any ? "r" : "0u") << ", h);\n";
                        break;
                    }
                }
                o << "  qsv::jit_rblock_split<" << K << ", " << NT << ", " << u32(op.fmask) << ", " << u32(op.tctrl)
                  << ", " << u32(m[0]) << ", " << u32(m[1]) << ", " << u32(m[2]) << ", " << u32(m[3]) << ", "
                  << u32(op.rot_tab) << ", " << S0 << ", " << S << ">(tile, [&](double2 (&v)[8], uint32_t r, uint32_t h) {\n";
                if (last > i) {
                    std::string call = o.str();
                    const std::string head = "  qsv::jit_rblock_split<";
                    const size_t at = call.rfind(head);
                    o.str("");
                    o << call.substr(0, at) << pre.str() << call.substr(at);
                }
                o << "    (void)r; (void)h;\n" << body.str();
                if (last > i) {
                    o << "  }, [&](double2& a, uint32_t idx) {\n    (void)idx;\n" << epi.str() << "  });\n";
                    i = last;
                } else {
                    o << "  }, qsv::NoEpi{});\n";
                }
                break;
            }
            // fold the pass relabel into this block's stores when it is the last op before it
            bool fold = false;
            std::string pmap;
            if (last + 1 == s.nops - 1 && ops[last + 1].kind == QSV_OP_RELABEL && op.xctrl == 0 && op.tctrl == 0 &&
                (1 << (K - __builtin_popcount(op.fmask))) == NT && env_int("QSV_JIT_FOLD_RELABEL", 1, 0, 1)) {
                const TileOp& rl = ops[last + 1];
                std::ostringstream pm;
                pm << "[](uint32_t x) { return 0u";
                for (int b = 0; b < K; ++b) {
                    const int dst = b < 8 ? rl.tpos[b] : rl.xbit[b - 8];
                    pm << " | (((x >> " << b << ") & 1u) << " << dst << ")";
                }
                pm << "; }";
                pmap = pm.str();
                fold = true;
            }
            o << "  qsv::jit_rblock<" << K << ", " << NT << ", " << KB << ", " << u32(op.fmask) << ", "
              << u32(op.tctrl) << ", " << u32(m[0]) << ", " << u32(m[1]) << ", " << u32(m[2]) << ", " << u32(m[3])
              << ", " << u32(op.rot_tab) << (fold ? ", true" : "") << ">(tile, [&](double2 (&v)[" << NV << "], uint32_t& r) {\n";
            if (last > i) {
                // hoisted constants must precede the call: re-emit the call after them
                std::string call = o.str();
                const std::string head = "  qsv::jit_rblock<";
                const size_t at = call.rfind(head);
                o.str("");
                o << call.substr(0, at) << pre.str() << call.substr(at);
            }
            o << "    (void)r;\n";
            const DevPrim* pr = reinterpret_cast<const DevPrim*>(blob + op.prim_byte);
            // Member rotation tracked through the body: register j holds member j ^ r.  A CX
            // whose control may be rotated swaps the pairs with register bit C = 1 (pure
            // renaming) and, on lanes whose rotation has bit C set, flips rotation bit T
            // instead of moving data (the complement set of pairs = all pairs composed with
            // these).  `rot` is the set of bits of r that may be non-zero at this point; the
            // host stores every U1/U2 matrix in all rotation variants.
            uint32_t rot = rot_any;
            const bool dyn_rot = env_int("QSV_JIT_DYNROT", 1, 0, 1) != 0;
            // Matrices of primitives whose slots are not rotated are emitted as literal
            // constants: the compiler folds them into constant-bank DFMA operands, saving the
            // SMEM loads and the registers that held them (QSV_JIT_LITERALS=0: from the blob)
            const bool literals = env_int("QSV_JIT_LITERALS", 1, 0, 1) != 0;
            int nlit = 0;
            auto lit = [&](const DevPrim& q, int n) {  // declares a local constant array, returns its name
                const double* d = reinterpret_cast<const double*>(blob + q.data_byte);
                const std::string name = "cm" + std::to_string(nlit++);
                std::ostringstream t;
                t << "    const double2 " << name << "[" << n << "] = {";
                char buf[96];
                for (int e = 0; e < n; ++e) {
                    std::snprintf(buf, sizeof(buf), "%s{%a, %a}", e ? ", " : "", d[2 * e], d[2 * e + 1]);
                    t << buf;
                }
                t << "};\n";
                o << t.str();
                return name;
            };
            for (int p = 0; p < op.nprim; ++p) {
                const DevPrim& q = pr[p];
                std::string mat = "reinterpret_cast<const double2*>(blob + " + std::to_string(q.data_byte) + ")";
                const bool ra = (rot >> q.a) & 1u, rb = (rot >> q.b) & 1u;
                if (literals) {
                    if ((q.kind == QSV_PRIM_U1 || q.kind == QSV_PRIM_U1R || q.kind == QSV_PRIM_U1I) && !ra)
                        mat = lit(q, 4);
                    else if (q.kind == QSV_PRIM_U2 && !ra && !rb)
                        mat = lit(q, 16);
                    else if (q.kind == QSV_PRIM_DIAG16 && rot == 0)
                        mat = lit(q, NV);
                }
                if (q.kind == QSV_PRIM_CX && ra && dyn_rot) {
                    o << "    qsv::rb_cx_plain<" << NV << ", " << int(q.a) << ", " << int(q.b) << ">(v);\n";
                    o << "    r ^= ((r >> " << int(q.a) << ") & 1u) << " << int(q.b) << ";\n";
                    rot |= 1u << q.b;
                    continue;
                }
                switch (q.kind) {
                case QSV_PRIM_U1:
                case QSV_PRIM_U1R:
                case QSV_PRIM_U1I: {
                    const char* fn = q.kind == QSV_PRIM_U1 ? "rb_u1" : (q.kind == QSV_PRIM_U1R ? "rb_u1r" : "rb_u1i");
                    o << "    qsv::" << fn << "<" << NV << ", " << int(q.a) << ">(v, " << mat;
                    if (ra)
                        o << " + 4u * ((r >> " << int(q.a) << ") & 1u)";
                    o << ");\n";
                    break;
                }
                case QSV_PRIM_U2:
                    o << "    qsv::rb_u2<" << NV << ", " << int(q.a) << ", " << int(q.b) << ">(v, " << mat;
                    if (ra || rb)
                        o << " + 16u * (((r >> " << int(q.a) << ") & 1u) | (((r >> " << int(q.b) << ") & 1u) << 1))";
                    o << ");\n";
                    break;
                case QSV_PRIM_CX:
                    if (ra)
                        o << "    qsv::rb_cx<" << NV << ", " << int(q.a) << ", " << int(q.b) << ">(v, r);\n";
                    else
                        o << "    qsv::rb_cx_plain<" << NV << ", " << int(q.a) << ", " << int(q.b) << ">(v);\n";
                    break;
                default:
                    o << "    qsv::rb_diag<" << NV << ">(v, " << mat << ", " << (rot ? "r" : "0u") << ");\n";
                    break;
                }
            }
            if (fold) {
                o << "  }, qsv::NoEpi{}, ";
                if (last > i)
                    o << "[&](double2 (&v)[" << NV << "], uint32_t base) {\n" << epib.str() << "  }";
                else
                    o << "qsv::NoEpiB{}";
                o << ", " << pmap << ");\n";
                i = last + 1;  // the fused diagonal ops and the relabel are done
            } else if (last > i) {
                o << "  }, qsv::NoEpi{}, [&](double2 (&v)[" << NV << "], uint32_t base) {\n" << epib.str() << "  });\n";
                i = last;  // the fused diagonal ops are done
            } else {
                o << "  });\n";
            }
            break;
        }
        default:
            o << "  // unknown op kind\n";
        }
        if (op.xctrl)
            o << "  }\n";
        o << "  }\n";
    }
    return o.str();
}

// Tile buffers / prefetch distance of the specialised kernels (QSV_TILE_NBUF,
// QSV_TILE_PD override the defaults for experiments).
int env_int(const char* name, int dflt, int lo, int hi) {
    const char* v = std::getenv(name);
    if (!v)
        return dflt;
    const int x = std::atoi(v);
    return x < lo ? lo : (x > hi ? hi : x);
}
int tile_nbuf() { return env_int("QSV_TILE_NBUF", kNumBuf, 2, 4); }
int tile_pd() { return env_int("QSV_TILE_PD", tile_nbuf() - 1, 1, tile_nbuf() - 1); }

std::string kernel_source(const std::string& name, int K, int minb, const std::string& body, int mt = 1) {
    std::ostringstream o;
    const int NT = threads_for_k(K);
    o << "extern \"C\" __global__ void __launch_bounds__(" << NT * mt << ", " << (mt > 1 ? 1 : minb) << ") " << name
      << "(double2* __restrict__ psi, const unsigned char* __restrict__ gblob, uint32_t blob_bytes,\n"
      << "    const __grid_constant__ qsv::GeomArg geom, uint64_t rank_base, uint64_t ntiles,\n"
      << "    const __grid_constant__ qsv::TmaDesc tmap) {\n"
      << "  qsv::pass_pipeline<" << K << ", " << NT << ", " << tile_nbuf() << ", " << tile_pd() << ", "
      << (env_int("QSV_TMA_SPREAD", 1, 0, 1) ? "true" : "false") << ", " << mt
      << ">(psi, gblob, blob_bytes, geom, rank_base, ntiles,\n"
      << "    [&](double2* tile, const unsigned char* blob, uint64_t full_base) {\n"
      << "  (void)full_base;\n"
      << body << "  }, &tmap);\n}\n";
    return o.str();
}

uint64_t fnv1a(const std::string& s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

std::string cache_dir() {
    if (const char* d = std::getenv("QSV_JIT_CACHE"))
        return d;
    const char* home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/qsv_jit";
}

void mkdirs(const std::string& p) {
    std::string cur;
    std::stringstream ss(p);
    std::string part;
    if (!p.empty() && p[0] == '/')
        cur = "/";
    while (std::getline(ss, part, '/')) {
        if (part.empty())
            continue;
        cur += part + "/";
        mkdir(cur.c_str(), 0755);
    }
}

// Compiles one translation unit to a cubin (or loads it from the cache).
const char* const kJitOpts[4] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-diag-suppress=177,550"};
std::string unit_cache_path(const std::string& src);

// Compiles one translation unit to a cubin (or loads it from the cache unless
// use_cache is false: a cached cubin the driver rejected is recompiled).
bool compile_unit(const std::string& src, std::vector<char>& cubin, std::string& err, bool use_cache = true) {
    if (const char* dump = std::getenv("QSV_JIT_DUMP")) {  // debugging: keep the generated source
        char name[64];
        std::snprintf(name, sizeof(name), "/qsv_%016llx.cu", static_cast<unsigned long long>(fnv1a(src)));
        std::ofstream(std::string(dump) + name) << src;
    }
    if (std::getenv("QSV_JIT_DRYRUN")) {  // diagnostics: count the kernels without compiling
        cubin.assign(1, 0);
        return true;
    }
    const std::string dir = cache_dir();
    const std::string path = unit_cache_path(src);
    if (use_cache) {
        std::ifstream in(path, std::ios::binary);
        if (in) {
            cubin.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
            if (!cubin.empty())
                return true;
        }
    }
    const Nvrtc& n = nvrtc();
    nvrtcProgram prog;
    static const char* opts[] = {kJitOpts[0], kJitOpts[1], kJitOpts[2], kJitOpts[3]};
    if (n.create(&prog, src.c_str(), "qsv_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        err = "nvrtcCreateProgram failed";
        return false;
    }
    const nvrtcResult rc = n.compile(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
    if (rc != NVRTC_SUCCESS) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        n.log(prog, log.data());
        err = "NVRTC compile failed: " + log.substr(0, 2000);
        n.destroy(&prog);
        return false;
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    cubin.resize(cs);
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    mkdirs(dir);
    // unique per process and thread (several ranks on one node share the cache);
    // only a completely written file is renamed into place
    std::ostringstream tn;
    tn << path << ".tmp." << getpid() << "." << std::this_thread::get_id();
    const std::string tmp = tn.str();
    bool good;
    {
        std::ofstream out(tmp, std::ios::binary);
        out.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
        out.flush();
        good = static_cast<bool>(out);
    }
    if (!good || std::rename(tmp.c_str(), path.c_str()) != 0)
        std::remove(tmp.c_str());  // the cache is an optimisation: the cubin in memory is fine
    return true;
}

std::string unit_cache_path(const std::string& src) {
    std::string key = src;
    for (const char* op : kJitOpts)
        key += op;
    char hex[32];
    std::snprintf(hex, sizeof(hex), "%016llx", static_cast<unsigned long long>(fnv1a(key)));
    return cache_dir() + "/qsv_" + hex + ".cubin";
}

} // namespace

bool jit_available(std::string& why) {
    if (!nvrtc().ok) {
        why = nvrtc().why;
        return false;
    }
    if (!driver().ok) {
        why = "CUDA driver entry points unavailable";
        return false;
    }
    return true;
}

namespace {

// Distinct pass structures of a program -> kernel sources (host only).
struct JitPlan {
    std::vector<std::string> bodies;
    std::vector<int> kernel_k, kernel_minb, kernel_mt, kernel_wide;
    std::vector<int> jit_of_step;
};

// A pass qualifies for wide kernels when every register block holds <= 8 amplitudes and no
// op needs a thread per 32-member group (dense k = 5).
bool wide_pass(const Step& s, const unsigned char* blob) {
    if (s.geom.K != 11 || split_blocks() || env_int("QSV_JIT_WIDE", 0, 0, 1) == 0)
        return false;
    const TileOp* ops = reinterpret_cast<const TileOp*>(blob);
    bool any_rb = false;
    for (int i = 0; i < s.nops; ++i) {
        if (ops[i].kind == QSV_OP_RBLOCK) {
            if (ops[i].k > 3)
                return false;
            any_rb = true;
        }
        if ((ops[i].kind == QSV_OP_DENSE && ops[i].k == 5) || ops[i].kind == QSV_OP_DMMA16)
            return false;
    }
    return any_rb;
}

// Dynamic SMEM of a specialised kernel: MT groups x NBUF tile buffers + the pass blob.
size_t jit_tile_smem(int K, int mt) { return sizeof(double2) * static_cast<size_t>(mt) * tile_nbuf() * (size_t{1} << K); }
constexpr size_t kSmemPerCta = 227 * 1024 - 4096;  // opt-in limit minus the static arrays

JitPlan plan_kernels_mode(const std::vector<Step>& steps, const unsigned char* host_blobs, int max_kernels,
                          bool class_mode);

// Fully specialised kernels (every structural quantity a constant) unless the program has
// more than QSV_JIT_CLASS_MIN distinct passes: then structure classes (masks, slots, tables
// and blob offsets read at run time, primitives through a rolled switch over the program's
// variants) share kernels.  Opt-in: UCCSD-28 drops from 4436 to 132 kernels, but the
// rolled bodies spill (48-164 B) and compile ~40x slower each, so NVRTC time does not
// improve (69 s vs ~47 s cold on the same 8 host cores; profiles/r02_kernel_ab.md).
JitPlan plan_kernels(const std::vector<Step>& steps, const unsigned char* host_blobs, int max_kernels) {
    const int class_min = env_int("QSV_JIT_CLASS_MIN", 1 << 30, 0, 1 << 30);
    JitPlan jp = plan_kernels_mode(steps, host_blobs, std::max(max_kernels, class_min + 1), false);
    if (static_cast<int>(jp.bodies.size()) <= class_min && static_cast<int>(jp.bodies.size()) <= max_kernels)
        return jp;
    return plan_kernels_mode(steps, host_blobs, max_kernels, true);
}

JitPlan plan_kernels_mode(const std::vector<Step>& steps, const unsigned char* host_blobs, int max_kernels,
                          bool class_mode) {
    JitPlan jp;
    std::vector<int> variants;
    if (class_mode) {
        for (const Step& s : steps) {
            if (s.desc.kind != QSV_STEP_PASS)
                continue;
            const unsigned char* blob = host_blobs + s.blob_off;
            const TileOp* ops = reinterpret_cast<const TileOp*>(blob);
            for (int i = 0; i < s.nops; ++i) {
                if (ops[i].kind != QSV_OP_RBLOCK)
                    continue;
                const DevPrim* pr = reinterpret_cast<const DevPrim*>(blob + ops[i].prim_byte);
                for (int p = 0; p < ops[i].nprim; ++p) {
                    const int key = (pr[p].kind << 4) | (pr[p].a << 2) | pr[p].b;
                    if (std::find(variants.begin(), variants.end(), key) == variants.end())
                        variants.push_back(key);
                }
            }
        }
        std::sort(variants.begin(), variants.end());
    }
    t_variants = class_mode ? &variants : nullptr;
    struct Reset {
        ~Reset() { t_variants = nullptr; }
    } reset;
    std::map<std::string, int> uniq;
    jp.jit_of_step.assign(steps.size(), -1);
    for (size_t i = 0; i < steps.size(); ++i) {
        const Step& s = steps[i];
        if (s.desc.kind != QSV_STEP_PASS || s.geom.K < 4)
            continue;
        int minb = 3;
        const bool wide = wide_pass(s, host_blobs + s.blob_off);
        t_wide = wide;
        struct WideReset {
            ~WideReset() { t_wide = false; }
        } wide_reset;
        int mt = wide ? 1 : jit_mt(s.geom.K);
        bool mt_ok = true;
        std::string body = gen_ops(s, host_blobs + s.blob_off, minb, mt, &mt_ok, class_mode);
        if (mt > 1 && (!mt_ok || jit_tile_smem(s.geom.K, mt) + s.blob_bytes > kSmemPerCta)) {
            mt = 1;
            body = gen_ops(s, host_blobs + s.blob_off, minb, 1, nullptr, class_mode);
        }
        const std::string key = std::to_string(s.geom.K) + "|" + std::to_string(minb) + "|" + std::to_string(mt) +
                                "|" + (wide ? "w|" : "|") + body;
        auto it = uniq.find(key);
        if (it == uniq.end()) {
            if (static_cast<int>(jp.bodies.size()) >= max_kernels)
                continue;  // beyond the budget: this pass keeps the interpreter
            it = uniq.emplace(key, static_cast<int>(jp.bodies.size())).first;
            jp.bodies.push_back(body);
            jp.kernel_k.push_back(s.geom.K);
            jp.kernel_minb.push_back(minb);
            jp.kernel_mt.push_back(mt);
            jp.kernel_wide.push_back(wide ? 1 : 0);
        }
        jp.jit_of_step[i] = it->second;
    }
    return jp;
}

// Kernels per NVRTC translation unit (QSV_JIT_UNIT overrides; every unit re-parses the
// device source, so larger units amortise it, smaller ones spread over more host threads)
int kernels_per_unit() { return env_int("QSV_JIT_UNIT", 6, 1, 256); }

// NVRTC-compiles the kernels of `jp` in translation units of kKernelsPerUnit,
// concurrently (no device needed).
bool compile_kernels(const JitPlan& jp, std::vector<std::vector<char>>& cubins, std::string& err,
                     std::vector<std::string>* sources = nullptr) {
    const int nk = static_cast<int>(jp.bodies.size());
    const int kKernelsPerUnit = kernels_per_unit();
    const int nunits = (nk + kKernelsPerUnit - 1) / kKernelsPerUnit;
    std::vector<std::string> srcs(nunits);
    for (int u = 0; u < nunits; ++u) {
        std::string src = kDeviceSource;
        for (int k = u * kKernelsPerUnit; k < std::min(nk, (u + 1) * kKernelsPerUnit); ++k) {
            t_wide = jp.kernel_wide[k] != 0;
            src += kernel_source("qsv_jit_" + std::to_string(k), jp.kernel_k[k], jp.kernel_minb[k], jp.bodies[k],
                                 jp.kernel_mt[k]);
            t_wide = false;
        }
        srcs[u] = std::move(src);
    }
    cubins.assign(nunits, {});
    std::vector<std::string> errs(nunits);
    std::vector<char> oks(nunits, 0);
    const int nthreads = std::max(1, std::min(nunits, static_cast<int>(std::thread::hardware_concurrency())));
    std::vector<std::thread> pool;
    for (int w = 0; w < nthreads; ++w)
        pool.emplace_back([&, w] {
            for (int u = w; u < nunits; u += nthreads)
                oks[u] = compile_unit(srcs[u], cubins[u], errs[u]) ? 1 : 0;
        });
    for (auto& t : pool)
        t.join();
    for (int u = 0; u < nunits; ++u)
        if (!oks[u]) {
            err = errs[u];
            return false;
        }
    if (sources)
        *sources = std::move(srcs);
    return true;
}

} // namespace

int jit_check(const std::vector<Step>& steps, const unsigned char* host_blobs, int max_kernels, int* kernels) {
    if (!nvrtc().ok) {
        set_error("qsv_program_jit_check: " + nvrtc().why);
        return QSV_E_STATE;
    }
    const JitPlan jp = plan_kernels(steps, host_blobs, max_kernels);
    std::vector<std::vector<char>> cubins;
    std::string err;
    if (!compile_kernels(jp, cubins, err)) {
        set_error("qsv_program_jit_check: " + err);
        return QSV_E_CUDA;
    }
    if (kernels)
        *kernels = static_cast<int>(jp.bodies.size());
    return QSV_OK;
}

struct JitBuild {
    std::vector<int> jit_of_step;
    std::vector<JitKernel> kernels;
    std::vector<void*> modules;  // CUmodule
    double seconds = 0;
    int rc = QSV_OK;
    std::string err;
};

namespace {

// Plans, compiles and loads the program's specialised kernels into `b`.  Reads only the
// program's immutable steps / blobs / device, so it can run on a background thread.
void jit_build(const qsv_program* prog, int max_kernels, JitBuild& b) {
    const auto t0 = std::chrono::steady_clock::now();
    auto fail = [&](int rc, const std::string& why) {
        const Driver& d = driver();
        for (void* m : b.modules)
            d.unload(static_cast<CUmodule>(m));
        b.modules.clear();
        b.kernels.clear();
        b.jit_of_step.assign(prog->steps.size(), -1);
        b.rc = rc;
        b.err = why;
    };
    std::string why;
    if (!jit_available(why))
        return fail(QSV_E_STATE, "qsv_program_jit: " + why);
    JitPlan jp = plan_kernels(prog->steps, prog->host_blobs.data(), max_kernels);
    b.jit_of_step = jp.jit_of_step;
    const int nk = static_cast<int>(jp.bodies.size());
    if (nk == 0)
        return;
    const int per_unit = kernels_per_unit();
    const int nunits = (nk + per_unit - 1) / per_unit;
    const std::vector<int>& kernel_k = jp.kernel_k;
    std::vector<std::vector<char>> cubins;
    std::vector<std::string> srcs;
    std::string err;
    if (!compile_kernels(jp, cubins, err, &srcs))
        return fail(QSV_E_CUDA, "qsv_program_jit: " + err);
    // load modules and functions
    const Driver& d = driver();
    cudaSetDevice(prog->ctx->device);
    cudaFree(nullptr);  // make sure the primary context is current (also on a background thread)
    b.kernels.assign(nk, {});
    for (int u = 0; u < nunits; ++u) {
        CUmodule mod;
        if (d.module_load(&mod, cubins[u].data()) != CUDA_SUCCESS) {
            // a stale or damaged cache entry: drop it and compile this unit afresh
            std::remove(unit_cache_path(srcs[u]).c_str());
            if (!compile_unit(srcs[u], cubins[u], err, false) || d.module_load(&mod, cubins[u].data()) != CUDA_SUCCESS)
                return fail(QSV_E_CUDA, "qsv_program_jit: cuModuleLoadData failed" +
                                            (err.empty() ? std::string() : ": " + err));
        }
        b.modules.push_back(mod);
        for (int k = u * per_unit; k < std::min(nk, (u + 1) * per_unit); ++k) {
            CUfunction f;
            const std::string name = "qsv_jit_" + std::to_string(k);
            if (d.get_function(&f, mod, name.c_str()) != CUDA_SUCCESS)
                return fail(QSV_E_CUDA, "qsv_program_jit: cuModuleGetFunction failed for " + name);
            const int K = kernel_k[k];
            const int mt = jp.kernel_mt[k];
            const size_t tile_smem = jit_tile_smem(K, mt);
            d.set_attr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                       static_cast<int>(std::min(tile_smem + kMaxBlobBytes, kSmemPerCta)));
            b.kernels[k].func = f;
            t_wide = jp.kernel_wide[k] != 0;
            b.kernels[k].nt = threads_for_k(K) * mt;
            t_wide = false;
            b.kernels[k].mt = mt;
            b.kernels[k].tile_smem = tile_smem;
        }
    }
    b.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Installs a successful build (host thread; no run of the program is being enqueued).
void jit_adopt(qsv_program* prog, JitBuild& b) {
    prog->jit_of_step = std::move(b.jit_of_step);
    prog->jit_kernels = std::move(b.kernels);
    for (void* m : b.modules)
        prog->jit_modules.push_back(m);
    b.modules.clear();
    for (auto& kv : prog->graphs)  // captured with the interpreter kernels
        cudaGraphExecDestroy(kv.second);
    prog->graphs.clear();
}

} // namespace

int jit_program(qsv_program* prog, int max_kernels, double* seconds) {
    if (int rc = jit_poll(prog, true); rc != QSV_OK)
        return rc;
    JitBuild b;
    jit_build(prog, max_kernels, b);
    if (b.rc != QSV_OK) {
        prog->jit_of_step.assign(prog->steps.size(), -1);
        set_error(b.err);
        return b.rc;
    }
    jit_adopt(prog, b);
    prog->jit_seconds = b.seconds;
    if (seconds)
        *seconds = b.seconds;
    return QSV_OK;
}

// Background compile: runs of the program use the interpreter kernel until the build is
// adopted by jit_poll (at the start of the next run), so the first result does not wait for
// NVRTC (UCCSD-28: ~170 s cold against a 16 s interpreted run).
int jit_start_async(qsv_program* prog, int max_kernels) {
    if (int rc = jit_poll(prog, true); rc != QSV_OK)
        return rc;
    for (const Step& s : prog->steps)
        if (s.desc.kind == QSV_STEP_PASS && s.geom.K > 11) {  // no interpreter to run them meanwhile
            double secs = 0;
            return jit_program(prog, max_kernels, &secs);
        }
    prog->jit_build = new JitBuild;
    prog->jit_done.store(false);
    prog->jit_thread = std::thread([prog, max_kernels] {
        jit_build(prog, max_kernels, *prog->jit_build);
        prog->jit_done.store(true, std::memory_order_release);
    });
    return QSV_OK;
}

bool jit_pending(const qsv_program* prog) { return prog->jit_build != nullptr; }

int jit_poll(qsv_program* prog, bool wait) {
    if (!prog->jit_build)
        return QSV_OK;
    if (!wait && !prog->jit_done.load(std::memory_order_acquire))
        return QSV_OK;
    prog->jit_thread.join();
    JitBuild* b = prog->jit_build;
    prog->jit_build = nullptr;
    int rc = b->rc;
    if (rc == QSV_OK) {
        cudaSetDevice(prog->ctx->device);
        // every launch enqueued so far used the interpreter; the adoption only changes later ones
        jit_adopt(prog, *b);
        prog->jit_seconds = b->seconds;
    } else {
        set_error(b->err);
    }
    delete b;
    return rc;
}

// Tensor map of a pass's tile on `st` (QSV_TMA_TENSOR=0 disables): the tile bits form
// runs of consecutive amplitude-index bits (the low run capped at 7 bits, others at 8, the
// box limit of 256 elements); each of the first five runs, with the non-tile bits above it,
// is one tensor dim whose box is the run; tile bits above the fifth run are iterated (at most
// 2^3 copies per tile).  Encoded once per (step, state buffer) and cached in the program.
void tile_tensor_map(const qsv_program* prog, const qsv_state* st, const Step& s, GeomArg& ga, TmaDesc& out) {
    static const bool on = env_int("QSV_TMA_TENSOR", 1, 0, 1) != 0;
    const Driver& d = driver();
    if (!on || !d.encode_tiled)
        return;
    const int L = s.geom.L, l = st->n_local;
    std::vector<int> bits;
    for (int b = 0; b < L; ++b)
        bits.push_back(b);
    for (int i = 0; i < s.geom.nhigh; ++i)
        bits.push_back(s.geom.high[i]);
    std::vector<std::pair<int, int>> runs;  // (start bit, length)
    for (int b : bits) {
        const int limit = runs.size() == 1 ? 7 : 8;  // the low run's box counts doubles
        if (!runs.empty() && runs.back().first + runs.back().second == b && runs.back().second < limit)
            ++runs.back().second;
        else
            runs.push_back({b, 1});
    }
    if (runs.empty() || runs[0].first != 0)
        return;
    const int rank = std::min<int>(5, static_cast<int>(runs.size()));
    std::vector<int> extra;
    for (size_t r = rank; r < runs.size(); ++r)
        for (int i = 0; i < runs[r].second; ++i)
            extra.push_back(runs[r].first + i);
    if (extra.size() > 3)
        return;  // more than 8 copies per tile: the per-run bulk copies are as good
    cuuint64_t gdim[5], gstride[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    uint32_t box_amps = 1;
    for (int dd = 0; dd < rank; ++dd) {
        const int lo = runs[dd].first;
        const int hi = dd + 1 < rank ? runs[dd + 1].first : l;
        if (hi - lo > 31)
            return;  // a tensor dim holds at most 2^32 elements
        gdim[dd] = (cuuint64_t{1} << (hi - lo)) * (dd == 0 ? 2 : 1);
        box[dd] = (1u << runs[dd].second) * (dd == 0 ? 2 : 1);
        box_amps <<= runs[dd].second;
        if (dd > 0)
            gstride[dd - 1] = (cuuint64_t{16} << lo);
        ga.tm_s[dd] = lo;
    }
    const auto key = std::make_pair(static_cast<const void*>(&s), static_cast<const void*>(st->amps));
    auto& cache = prog->tmaps;
    auto it = cache.find(key);
    if (it == cache.end()) {
        CUtensorMap tm;
        if (d.encode_tiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank), st->amps, gdim,
                           gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return;
        static_assert(sizeof(CUtensorMap) == sizeof(TmaDesc), "tensor map size");
        TmaDesc t;
        std::memcpy(&t, &tm, sizeof(t));
        it = cache.emplace(key, t).first;
    }
    out = it->second;
    ga.tm_rank = rank;
    ga.tm_nx = static_cast<int32_t>(extra.size());
    for (size_t i = 0; i < extra.size(); ++i)
        ga.tm_x[i] = extra[i];
    ga.tm_box_amps = box_amps;
}

cudaError_t launch_jit(const qsv_program* prog, const qsv_state* st, size_t step, const unsigned char* d_blob,
                       uint64_t rank_base, cudaStream_t stream, const LaunchRange& rg) {
    const Step& s = prog->steps[step];
    const JitKernel& jk = prog->jit_kernels[prog->jit_of_step[step]];
    const size_t smem = jk.tile_smem + s.blob_bytes;
    int per_sm = 0;
    const Driver& d = driver();
    if (d.occupancy(&per_sm, static_cast<CUfunction>(jk.func), jk.nt, smem) != CUDA_SUCCESS || per_sm < 1)
        per_sm = 1;
    GeomArg ga{};
    ga.L = s.geom.L;
    ga.nhigh = s.geom.nhigh;
    for (int i = 0; i < s.geom.nhigh; ++i)
        ga.high[i] = s.geom.high[i];
    {
        static const int poison = [] {
            const char* e = std::getenv("QSV_DEBUG_POISON");
            return e && e[0] == '1' ? 1 : 0;
        }();
        ga.poison = poison;
    }
    if (rg.fuse) {
        ga.peer = rg.fuse->peer;
        ga.flag_mine = rg.fuse->flag_mine;
        ga.flag_peer = rg.fuse->flag_peer;
        ga.epoch = rg.fuse->epoch;
        ga.sv = rg.fuse->sv;
        ga.sv_tile = rg.fuse->sv_tile;
        ga.sv_tidx = rg.fuse->sv_tidx;
        ga.sgbit = rg.fuse->sgbit;
        ga.spush = rg.fuse->push;
    }
    const uint64_t all_tiles = st->size >> s.geom.K;
    const uint64_t region_tiles = apply_region(ga, rg, all_tiles);
    ga.tile0 = std::min(rg.tile0, region_tiles);
    const uint64_t tiles = std::min(rg.count, region_tiles - ga.tile0);
    if (tiles == 0)
        return cudaSuccess;
    const int sms = rg.sms > 0 ? std::min(rg.sms, st->ctx->sm_count) : st->ctx->sm_count;
    const uint64_t ctas_needed = (tiles + jk.mt - 1) / jk.mt;
    uint64_t grid = std::min<uint64_t>(ctas_needed, static_cast<uint64_t>(per_sm) * sms);
    if (const char* g = std::getenv("QSV_DEBUG_GRID"))  // debug: fewer persistent CTAs, other tile order
        grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, std::strtoull(g, nullptr, 10)));
    if (rg.fuse)  // one flag per CTA (kFlagBytes)
        grid = std::min<uint64_t>(grid, kFlagBytes / sizeof(unsigned long long));
    double2* psi = st->amps;
    uint32_t bb = s.blob_bytes;
    uint64_t rb = rank_base, nt = tiles;
    TmaDesc tmap{};
    ga.tm_rank = 0;
    if (!rg.fuse && ga.nreg == 0 && jk.mt == 1)
        tile_tensor_map(prog, st, s, ga, tmap);
    void* args[] = {&psi, const_cast<unsigned char**>(&d_blob), &bb, &ga, &rb, &nt, &tmap};
    const CUresult r = d.launch(static_cast<CUfunction>(jk.func), static_cast<unsigned>(grid), 1, 1,
                                static_cast<unsigned>(jk.nt), 1, 1, static_cast<unsigned>(smem),
                                reinterpret_cast<CUstream>(stream), args, nullptr);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

void jit_release(qsv_program* prog) {
    if (prog->jit_build) {  // a background compile still running: wait, then drop its modules
        prog->jit_thread.join();
        const Driver& d = driver();
        for (void* m : prog->jit_build->modules)
            d.unload(static_cast<CUmodule>(m));
        delete prog->jit_build;
        prog->jit_build = nullptr;
    }
    if (prog->jit_modules.empty())
        return;
    const Driver& d = driver();
    for (void* m : prog->jit_modules)
        d.unload(static_cast<CUmodule>(m));
    prog->jit_modules.clear();
}

} // namespace qsv
