// Blackwell packed fp32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2).
//
// A pair lives in one 64-bit register pair; PTX add/sub/mul/fma.rn.f32x2
// round each element to nearest exactly as the scalar instruction would, so
// code written on pairs computes the same bits as the same code on scalars.
// Uniform operands go in through dup2(), which ptxas folds into the .F32
// broadcast operand selector (no moves).
#pragma once

#include <cuda_runtime.h>

namespace ubs {

using f32x2 = unsigned long long;

__device__ __forceinline__ f32x2 pk2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 up2(f32x2 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f32x2 dup2(float a) { return pk2(a, a); }
// in-place forms for loop-carried pairs (a fresh "=l" output would cost a
// register-pair copy per visit)
__device__ __forceinline__ void fma2_acc(f32x2 &c, f32x2 a, f32x2 b) {  // c = a b + c
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}
__device__ __forceinline__ void fma2_scale(f32x2 &c, f32x2 a, f32x2 b) {  // c = a c + b (== c a + b)
    // the accumulator as the B operand: with it as A, ptxas computes into a
    // fresh pair and copies every loop-carried pair back (10 MOVs per visit)
    asm("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(c) : "l"(a), "l"(b));
}
__device__ __forceinline__ void sub2_acc(f32x2 &c, f32x2 a) {  // c = c - a
    asm("sub.rn.f32x2 %0, %0, %1;" : "+l"(c) : "l"(a));
}

}  // namespace ubs
