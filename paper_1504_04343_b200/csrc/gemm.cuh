// gemm.cuh -- host-side description of one lowered GEMM (replaces convlow::multiply,
// gemm.cpp:93-122) executed by the tcgen05 3xTF32 kernel in gemm.cu.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace cct {

// How an operand is stored in global memory (row-major, leading dim `ld` floats):
//   KMaj  : rows are the M (or N) index, columns the reduction index K
//   MNMaj : rows are the reduction index K, columns the M (or N) index
enum class Major : int { K = 0, MN = 1 };

struct Operand {
    const float* ptr = nullptr;
    int64_t ld = 0;  // floats; must be a multiple of 4 (16-byte TMA strides)
    Major major = Major::K;
};

// Epilogue address map: element (row m, col n) of split s goes to
//   ptr + (m / mdiv) * s_mq + (m % mdiv) * s_mr + (n / ndiv) * s_nq + (n % ndiv) * s_n + s * s_split
// (row = TMEM lane; s_mr == 1 gives fully coalesced stores).
struct OutMap {
    float* ptr = nullptr;
    int64_t mdiv = INT64_MAX;
    int64_t s_mq = 0, s_mr = 1, s_n = 0, s_split = 0;
    int64_t ndiv = INT64_MAX, s_nq = 0;
    int64_t mlim = INT64_MAX;  // rows with (m % mdiv) >= mlim are not stored (padded channels)
    int64_t nmlim = INT64_MAX; // columns with (n % ndiv) >= nmlim are not stored (two-level map only)
    // fused epilogue (final stores only): v = act(v + bias[n]), act = ReLU when relu != 0
    const float* bias = nullptr;
    int relu = 0;
    // transposing epilogue: rows of the output are contiguous along n (e.g. NCHW y of a
    // swapped GEMM, rows = channels); the bias is then indexed by the ROW.  Needs K-major
    // A and B, no CTA pairs, BN >= 192 (run_gemm forces those)
    int transposed = 0;
};

// Implicit Type 1 lowering: operand A is read straight from the NHWC input x
// through a TMA im2col tensor map (no Dhat in HBM).  Row (or K) index = output
// pixel (q, r, c); lowered column = (i, j, ch) with ch fastest -- the same order
// as the materialised Dhat, so B (the KernelBank) is unchanged.
//   A.major == K  (forward; backward-data = forward of dy (NHWC) with rotated
//                  weights): tile = 128 pixels x 16 channels of one tap
//   A.major == MN (backward-weight): tile = 16 pixels x (4 x 32 channels)
// Channels per tap in the lowered index are dk (0: = d).  An MN-major A needs
// whole 32-channel boxes per tap, so a layer with d % 32 != 0 uses dk = d rounded
// up to 32: the boxes read past channel d-1 are zero-filled by TMA and the
// epilogue skips those rows (OutMap::mlim).
struct Im2col {
    const float* x = nullptr;  // nullptr: A is an ordinary (materialised) matrix
    int64_t b = 0, n = 0, d = 0, k = 0, s = 1, p = 0, m = 0;
    int64_t dk = 0;
    int64_t cs = 0;  // channel stride of a pixel in x (0: = d); > d reads one channel group
    // 0: A = im2col(x) (M = pixels, or MN-major for backward-weight); 1: B = im2col(x) (N =
    // pixels, K-major: swapped forward / backward-data); 2: B = MN-major im2col(x) (N = (tap,
    // channel), K = pixels: swapped backward-weight of a narrow bank)
    int operand = 0;
};

struct GemmProblem {
    int64_t M = 0, N = 0, K = 0;
    Operand A, B;
    OutMap C;
    int splits = 1;  // split-K factor; each split writes its own slice (s_split)
    int chain2 = 0;  // two accumulation chains in TMEM (K halves) summed in the epilogue
                     // instead of a 2-way split-K (K-major operands, tile width >= 192)
    int passes = 3;  // 3 = 3xTF32 (fp32-accurate), 1 = plain TF32 (diagnostic only)
    int bn = 0;      // 0 = choose
    Im2col im2col;   // implicit lowering of A (Type 1)
    // scratch for stream-K partial tiles (gemm_workspace_bytes); without it the
    // kernel runs data-parallel whole tiles
    void* ws = nullptr;
    size_t ws_bytes = 0;
};

// scratch run_gemm can use for this problem (0: none needed)
size_t gemm_workspace_bytes(const GemmProblem& g);

// Can this layer use the implicit (im2col) A operand?  d % 16 == 0 (one TMA box
// never straddles a filter tap; backward-weight pads the tap to im2col_dk).
bool im2col_ok(int64_t d, bool mn_major);
// channels per tap of the lowered index for an im2col A operand
int64_t im2col_dk(int64_t d, bool mn_major);

// Tile constants shared by the launcher and the kernel.
constexpr int kBM = 128;
constexpr int kBK = 16;
// longest single TMEM accumulation chain, in k-blocks (= 4096 reduction terms)
constexpr int kMaxChainKB = 256;

int choose_bn(int64_t N);
// split-K factor: at least the accuracy floor (chains <= kMaxChainKB k-blocks),
// then the count whose (pair-)units fill the last wave best
int choose_splits(int64_t M, int64_t N, int64_t K, int num_sms, int bn, int cg, int chains = 1);
// the same for a concrete problem (tile width and CTA-pair mode as run_gemm picks them);
// the count that actually runs (no empty split)
int plan_splits(const GemmProblem& g);
// splits that run when s are requested over kb k-blocks (empty trailing splits dropped)
int effective_splits(int64_t kb, int s);
// tile width the kernel uses for a problem
int tile_n(const GemmProblem& g);

cudaError_t run_gemm(const GemmProblem& g, cudaStream_t stream);

}  // namespace cct
