// op_costs.cu — SASS cost of each algorithmic operation of the k-NN search as the
// product kernel (paper_2111_04182_b200/csrc/knn.cu, 3D fp32 path) implements it.
// Each kernel runs one operation per loop iteration (#pragma unroll 1) on inputs in
// shared memory; scripts/op_costs.py counts the SASS instructions of each loop body
// (cuobjdump -sass) minus the loop overhead and writes profiles/rNN_op_costs.json.
// The expressions are the product's (same operand order and rounding modes).
#include <cstdint>
#include <cuda_runtime.h>

// distance test, uniform pass: 4 staged candidates per step, packed f32x2 (knn.cu scan_span)
extern "C" __global__ void op_dist4(const float* __restrict__ in, float wb, int iters, uint32_t* out) {
    __shared__ __align__(16) float fx[64], fy[64], fz[64];
    if (threadIdx.x < 64) { fx[threadIdx.x] = in[threadIdx.x]; fy[threadIdx.x] = in[64 + threadIdx.x]; fz[threadIdx.x] = in[128 + threadIdx.x]; }
    __syncthreads();
    const float q0 = in[threadIdx.x], q1 = in[threadIdx.x + 1], q2 = in[threadIdx.x + 2];
    const float2 qx = make_float2(q0, q0), qy = make_float2(q1, q1), qz = make_float2(q2, q2);
    uint32_t hit = 0;
#pragma unroll 1
    for (int j0 = 0; j0 < iters; j0 += 4) {
        const int j = j0 & 60;
        const float4 X = *reinterpret_cast<const float4*>(&fx[j]);
        const float4 Y = *reinterpret_cast<const float4*>(&fy[j]);
        const float4 Z = *reinterpret_cast<const float4*>(&fz[j]);
        const float2 dx0 = __fadd2_rn(qx, make_float2(-X.x, -X.y)), dx1 = __fadd2_rn(qx, make_float2(-X.z, -X.w));
        const float2 dy0 = __fadd2_rn(qy, make_float2(-Y.x, -Y.y)), dy1 = __fadd2_rn(qy, make_float2(-Y.z, -Y.w));
        const float2 dz0 = __fadd2_rn(qz, make_float2(-Z.x, -Z.y)), dz1 = __fadd2_rn(qz, make_float2(-Z.z, -Z.w));
        const float2 s0 = __ffma2_rn(dz0, dz0, __ffma2_rn(dy0, dy0, __fmul2_rn(dx0, dx0)));
        const float2 s1 = __ffma2_rn(dz1, dz1, __ffma2_rn(dy1, dy1, __fmul2_rn(dx1, dx1)));
        const uint32_t hb = (s0.x <= wb ? 1u : 0u) | (s0.y <= wb ? 2u : 0u) | (s1.x <= wb ? 4u : 0u) | (s1.y <= wb ? 8u : 0u);
        hit |= hb << (j0 & 28);
    }
    out[threadIdx.x] = hit;
}

// the same test as the final kernel runs it (ZD_SIGNMASK): the sign bit of wb - d2 of
// each candidate is funnel-shifted into the miss mask
extern "C" __global__ void op_dist4_final(const float* __restrict__ in, float wb, int iters, uint32_t* out) {
    __shared__ __align__(16) float fx[64], fy[64], fz[64];
    if (threadIdx.x < 64) { fx[threadIdx.x] = in[threadIdx.x]; fy[threadIdx.x] = in[64 + threadIdx.x]; fz[threadIdx.x] = in[128 + threadIdx.x]; }
    __syncthreads();
    const float q0 = in[threadIdx.x], q1 = in[threadIdx.x + 1], q2 = in[threadIdx.x + 2];
    const float2 qx = make_float2(q0, q0), qy = make_float2(q1, q1), qz = make_float2(q2, q2);
    const float2 wb2 = make_float2(wb, wb);
    uint32_t miss = 0;
#pragma unroll 1
    for (int j0 = 0; j0 < iters; j0 += 4) {
        const int j = j0 & 60;
        const float4 X = *reinterpret_cast<const float4*>(&fx[j]);
        const float4 Y = *reinterpret_cast<const float4*>(&fy[j]);
        const float4 Z = *reinterpret_cast<const float4*>(&fz[j]);
        const float2 dx0 = __fadd2_rn(qx, make_float2(-X.x, -X.y)), dx1 = __fadd2_rn(qx, make_float2(-X.z, -X.w));
        const float2 dy0 = __fadd2_rn(qy, make_float2(-Y.x, -Y.y)), dy1 = __fadd2_rn(qy, make_float2(-Y.z, -Y.w));
        const float2 dz0 = __fadd2_rn(qz, make_float2(-Z.x, -Z.y)), dz1 = __fadd2_rn(qz, make_float2(-Z.z, -Z.w));
        const float2 s0 = __ffma2_rn(dz0, dz0, __ffma2_rn(dy0, dy0, __fmul2_rn(dx0, dx0)));
        const float2 s1 = __ffma2_rn(dz1, dz1, __ffma2_rn(dy1, dy1, __fmul2_rn(dx1, dx1)));
        const float2 m0 = __fadd2_rn(wb2, make_float2(-s0.x, -s0.y));
        const float2 m1 = __fadd2_rn(wb2, make_float2(-s1.x, -s1.y));
        asm("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(miss) : "r"(__float_as_uint(m0.x)));
        asm("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(miss) : "r"(__float_as_uint(m0.y)));
        asm("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(miss) : "r"(__float_as_uint(m1.x)));
        asm("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(miss) : "r"(__float_as_uint(m1.y)));
    }
    out[threadIdx.x] = miss;
}

// box test of one child box (knn.cu box_dist / gap_d2 + within, 3D fp32)
extern "C" __global__ void op_box(const float* __restrict__ in, float wb, int iters, uint32_t* out) {
    __shared__ float b[6 * 64];
    for (int t = threadIdx.x; t < 6 * 64; t += blockDim.x) b[t] = in[t];
    __syncthreads();
    const float q0 = in[threadIdx.x], q1 = in[threadIdx.x + 1], q2 = in[threadIdx.x + 2];
    const float qf[3] = {q0, q1, q2};
    uint32_t acc = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        const float* bx = b + 6 * (i & 63);
        // the product's gap_d2: per axis one 3-input max, max(lo - q, q - hi, 0) (FMNMX3)
        float t[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float r;
            asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(bx[a] - qf[a]), "f"(qf[a] - bx[3 + a]), "f"(0.f));
            t[a] = r;
        }
        const float df = fmaf(t[2], t[2], fmaf(t[1], t[1], t[0] * t[0]));
        acc += df <= wb ? 1u : 0u;
    }
    out[threadIdx.x] = acc;
}

// one k-best insertion on the hit path (knn.cu scan_span hit loop: next hit bit, the
// candidate's fp32 d2, self test, ru(d2), the branch-free median insertion into the
// K = 10 list, the new bound, the buffer append)
extern "C" __global__ void op_insert(const float* __restrict__ in, int iters, uint32_t hitmask, uint2* out) {
    __shared__ float fx[32], fy[32], fz[32];
    __shared__ int32_t fid[32], fp[32];
    __shared__ int2 be[32][32];
    if (threadIdx.x < 32) { fx[threadIdx.x] = in[threadIdx.x]; fy[threadIdx.x] = in[32 + threadIdx.x]; fz[threadIdx.x] = in[64 + threadIdx.x];
                            fid[threadIdx.x] = (int)in[96 + threadIdx.x]; fp[threadIdx.x] = threadIdx.x; }
    __syncthreads();
    const float q0 = in[threadIdx.x], q1 = in[threadIdx.x + 1], q2 = in[threadIdx.x + 2];
    const int32_t qid = threadIdx.x;
    const int lane = threadIdx.x & 31;
    float fa[10];
#pragma unroll
    for (int t = 0; t < 10; ++t) fa[t] = in[200 + t];
    float wb = fa[9];
    int cnt = 0;
    uint32_t hit = hitmask;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        if (!hit) hit = hitmask;
        const int j = __ffs(hit) - 1;
        hit &= hit - 1;
        const float dx = q0 - fx[j], dy = q1 - fy[j], dz = q2 - fz[j];
        const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        if (fid[j] == qid) continue;
        if (df > wb) continue;
        const float xf = __fmul_ru(df, 1.0f + 0x1p-21f);
#pragma unroll
        for (int t = 9; t > 0; --t) fa[t] = fmaxf(fa[t - 1], fminf(fa[t], xf));
        fa[0] = fminf(fa[0], xf);
        wb = __fmul_ru(fa[9], 1.0f + 0x1p-21f);
        be[cnt & 31][lane] = make_int2(fp[j], __float_as_int(xf));
        cnt = (cnt + 1) & 31;
    }
    out[threadIdx.x] = make_uint2(__float_as_uint(wb), cnt + be[lane][lane].x);
}

// the same insertion as the final kernel runs it (ZD_FA_BF16): the K = 10 list as five
// packed bf16 pairs rounded up (PRMT + 2 HMNMX2 per pair)
extern "C" __global__ void op_insert_final(const float* __restrict__ in, int iters, uint32_t hitmask, uint2* out) {
    __shared__ float fx[32], fy[32], fz[32];
    __shared__ int32_t fid[32], fp[32];
    __shared__ int2 be[32][32];
    if (threadIdx.x < 32) { fx[threadIdx.x] = in[threadIdx.x]; fy[threadIdx.x] = in[32 + threadIdx.x]; fz[threadIdx.x] = in[64 + threadIdx.x];
                            fid[threadIdx.x] = (int)in[96 + threadIdx.x]; fp[threadIdx.x] = threadIdx.x; }
    __syncthreads();
    const float q0 = in[threadIdx.x], q1 = in[threadIdx.x + 1], q2 = in[threadIdx.x + 2];
    const int32_t qid = threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t p[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) p[t] = __float_as_uint(in[200 + t]);
    float wb = __uint_as_float(p[4] & 0xffff0000u);
    int cnt = 0;
    uint32_t hit = hitmask;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        if (!hit) hit = hitmask;
        const int j = __ffs(hit) - 1;
        hit &= hit - 1;
        const float dx = q0 - fx[j], dy = q1 - fy[j], dz = q2 - fz[j];
        const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        if (fid[j] == qid) continue;
        if (df > wb) continue;
        const float xf = __fmul_ru(df, 1.0f + 0x1p-21f);
        uint32_t x;
        asm("prmt.b32 %0, %1, 0, 0x3232;" : "=r"(x) : "r"(__float_as_uint(xf) + 0xffffu));
        uint32_t sh[5];
        sh[0] = p[0] << 16;
#pragma unroll
        for (int t = 1; t < 5; ++t) asm("prmt.b32 %0, %1, %2, 0x5432;" : "=r"(sh[t]) : "r"(p[t - 1]), "r"(p[t]));
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            uint32_t m;
            asm("min.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(p[t]), "r"(x));
            asm("max.bf16x2 %0, %1, %2;" : "=r"(p[t]) : "r"(sh[t]), "r"(m));
        }
        wb = __fmul_ru(__uint_as_float(p[4] & 0xffff0000u), 1.0f + 0x1p-21f);
        be[cnt & 31][lane] = make_int2(fp[j], __float_as_int(xf));
        cnt = (cnt + 1) & 31;
    }
    out[threadIdx.x] = make_uint2(__float_as_uint(wb), cnt + be[lane][lane].x);
}

// Alg. 3 stop test at one ascent (knn.cu lane_stop, 3D fp32)
extern "C" __global__ void op_ascent(const float* __restrict__ in, int iters, uint32_t* out) {
    __shared__ float b[6 * 64];
    for (int t = threadIdx.x; t < 6 * 64; t += blockDim.x) b[t] = in[t];
    __syncthreads();
    const float q0 = in[threadIdx.x], q1 = in[threadIdx.x + 1], q2 = in[threadIdx.x + 2];
    const float qf[3] = {q0, q1, q2};
    const float bound = in[400];
    uint32_t acc = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        const float* bx = b + 6 * (i & 63);
        float m = INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a) m = fminf(m, fminf(qf[a] - bx[a], bx[3 + a] - qf[a]));
        const float mm = m + 1.0f;
        acc += (m >= 0.f && __fmul_rd(mm, mm) > bound) ? 1u : 0u;
    }
    out[threadIdx.x] = acc;
}
