// stage_variants.cuh -- stage schedules measured and REJECTED by the stage bench (csrc/stage_bench.cu,
// profiles/README.md): kept so the A/B history can be re-run, never included by the product kernels.
// The product schedules are in zhang_step.cuh (conv2_back V14 fast / V15 EXACT, C1 gradient beside g_k2).
#pragma once

#include "zhang_step.cuh"

namespace tlb {

__device__ __forceinline__ void stage_pool2(const Smem& s) {

  for (int t = threadIdx.x; t < 192; t += blockDim.x) {
    const int c = t >> 4, py = (t >> 2) & 3, px = t & 3;
    const float* q = s.c2 + (c * 8 + 2 * py) * 8 + 2 * px;
    s.s2[t] = fmul(fadd(fadd(fadd(q[0], q[1]), q[8]), q[9]), 0.25f);
  }
}

// backin d_s1 = sum_i backin(dz2[i], k2[i], s1), then backavgpool + backsigmoid through c1 -> dz1.
//
// One lane per item (channel c, output rows p0 = 2pp and p0+1, columns 4qq..4qq+3) runs all twelve
// kernels in order.  Per kernel it holds the 25 weights in registers and streams the six padded dz2
// rows its two output rows need, so each loaded row feeds both rows' taps; lanes of a warp share the
// dz2 rows (broadcast) across channels, which keeps shared-memory traffic ~4x below per-row tiling.
// The reference's clipped nested sums (nn.cpp:169-189: per i, row sums over u2 from 0, outer sum over
// u1 from 0, then acc = acc + term over i as network.cpp:135-138) only ever see padded zero products
// prepended or appended to a row/outer sum, and x + (+-0) == x (with +0 + -0 == +0), so EXACT stays
// bit-identical.  Fast mode accumulates every tap with FFMA.
// backin term of kernel i for the 2x4 output tile (p0.., 4qq..): ordered nested sums (EXACT) into
// b[orow][o], or FFMA accumulation straight into acc (fast).
template <bool EXACT>
__device__ __forceinline__ void backin_kernel_term(const Smem& s, int i, int c, int p0, int qq, float (&b)[2][4],
                                                   float (&acc)[2][4]) {
  float w[5][5];
#pragma unroll
  for (int u1 = 0; u1 < 5; ++u1) {
    const float4* wp = reinterpret_cast<const float4*>(s.Kp + ((i * 6 + c) * 5 + u1) * 8);
    const float4 w0 = wp[0], w1 = wp[1];
    w[u1][0] = w0.x; w[u1][1] = w0.y; w[u1][2] = w0.z; w[u1][3] = w0.w; w[u1][4] = w1.x;
  }
#pragma unroll
  for (int orow = 0; orow < 2; ++orow)
#pragma unroll
    for (int o = 0; o < 4; ++o) b[orow][o] = 0.0f;
  // padded rows R = p0 + rr, rr = 5..0: output row orow uses tap row u1 = orow + 4 - rr (ascending)
#pragma unroll
  for (int rr = 5; rr >= 0; --rr) {
    const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, p0 + rr, 4 * qq));
    const float4 d0 = dp[0], d1 = dp[1];
    const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
    for (int orow = 0; orow < 2; ++orow) {
      const int u1 = orow + 4 - rr;
      if (u1 < 0 || u1 > 4) continue;
      if constexpr (EXACT) {
        float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int u2 = 0; u2 < 5; ++u2)
#pragma unroll
          for (int o = 0; o < 4; ++o) rs[o] = mac<true>(rs[o], w[u1][u2], d[o - u2 + 4]);
#pragma unroll
        for (int o = 0; o < 4; ++o) b[orow][o] = fadd(b[orow][o], rs[o]);
      } else {
#pragma unroll
        for (int u2 = 0; u2 < 5; ++u2)
#pragma unroll
          for (int o = 0; o < 4; ++o) acc[orow][o] = __fmaf_rn(w[u1][u2], d[o - u2 + 4], acc[orow][o]);
      }
    }
  }
}

// backavgpool (x0.25) + backsigmoid through c1 for the 4x8 block of c1 owned by a backin tile.
__device__ __forceinline__ void backin_to_dz1(const Smem& s, int c, int p0, int qq, const float (&acc)[2][4]) {
#pragma unroll
  for (int orow = 0; orow < 2; ++orow)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      float4* cp = reinterpret_cast<float4*>(s.c1 + c1_at(c, 2 * (p0 + orow) + dy, 8 * qq));
      const float4 v0 = cp[0], v1 = cp[1];
      float cv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const float dc = fmul(acc[orow][x >> 1], 0.25f);
        cv[x] = fmul(fmul(dc, cv[x]), fsub(1.0f, cv[x]));
      }
      cp[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
      cp[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
    }
}

// backin d_s1 = sum_i backin(dz2[i], k2[i], s1), then backavgpool + backsigmoid through c1 -> dz1.
//
// Item = (channel c, output rows p0 = 2pp and p0+1, columns 4qq..4qq+3); NSPLIT lanes share an item,
// lane `part` running kernels [part*12/NSPLIT, (part+1)*12/NSPLIT).  Per kernel a lane holds the 25
// weights in registers and streams the six padded dz2 rows the two output rows need, so each loaded
// row feeds both rows' taps; lanes of a warp share the dz2 rows (broadcast) across channels.
// The reference's clipped nested sums (nn.cpp:169-189: per i, row sums over u2 from 0, outer sum over
// u1 from 0, then acc = acc + term over i as network.cpp:135-138) only ever see padded zero products
// prepended or appended to a row/outer sum, and x + (+-0) == x (with +0 + -0 == +0), so EXACT stays
// bit-identical; with NSPLIT = 2 the second lane's six per-kernel terms reach the first lane by
// shuffle, in kernel order.  Fast mode accumulates every tap with FFMA and combines with one xor.
template <bool EXACT, int NSPLIT>
__device__ __forceinline__ void backin_tile(const Smem& s, int lane_item, bool valid) {
  const int item = valid ? lane_item / NSPLIT : 0, part = lane_item % NSPLIT;
  const int c = item / 18, rem = item - c * 18, pp = rem / 3, qq = rem - pp * 3, p0 = 2 * pp;
  constexpr int KPL = 12 / NSPLIT;  // kernels per lane
  float acc[2][4];
#pragma unroll
  for (int orow = 0; orow < 2; ++orow)
#pragma unroll
    for (int o = 0; o < 4; ++o) acc[orow][o] = 0.0f;
  if constexpr (NSPLIT == 1) {
#pragma unroll 1
    for (int i = 0; i < 12; ++i) {
      float b[2][4];
      backin_kernel_term<EXACT>(s, i, c, p0, qq, b, acc);
      if constexpr (EXACT) {
#pragma unroll
        for (int orow = 0; orow < 2; ++orow)
#pragma unroll
          for (int o = 0; o < 4; ++o) acc[orow][o] = fadd(acc[orow][o], b[orow][o]);
      }
    }
  } else {
    float mine[KPL][2][4];
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      backin_kernel_term<EXACT>(s, part * KPL + k, c, p0, qq, mine[k], acc);
      if constexpr (EXACT) {
        if (part == 0) {
#pragma unroll
          for (int orow = 0; orow < 2; ++orow)
#pragma unroll
            for (int o = 0; o < 4; ++o) acc[orow][o] = fadd(acc[orow][o], mine[k][orow][o]);
        }
      }
    }
    if constexpr (EXACT) {
#pragma unroll
      for (int k = 0; k < KPL; ++k)
#pragma unroll
        for (int orow = 0; orow < 2; ++orow)
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const float v = __shfl_xor_sync(0xffffffffu, mine[k][orow][o], 1);
            acc[orow][o] = fadd(acc[orow][o], v);
          }
    } else {
#pragma unroll
      for (int orow = 0; orow < 2; ++orow)
#pragma unroll
        for (int o = 0; o < 4; ++o) acc[orow][o] += __shfl_xor_sync(0xffffffffu, acc[orow][o], 1);
    }
  }
  if (valid && part == 0) backin_to_dz1(s, c, p0, qq, acc);
}

template <bool EXACT>
__device__ __forceinline__ void backin_item(const Smem& s, int item) {
  backin_tile<EXACT, 1>(s, item, true);
}

// backin variant: lane quads split the twelve kernels 3 per lane; EXACT hands the per-kernel terms to
// lane 0 of the quad by shuffle so the ordered chain over i stays on one lane.
template <bool EXACT>
__device__ __forceinline__ void backin_quad(const Smem& s, int lane_item, bool valid) {
  const int item = valid ? lane_item >> 2 : 0, q4 = lane_item & 3;
  const int c = item / 18, rem = item - c * 18, pp = rem / 3, qq = rem - pp * 3, p0 = 2 * pp;
  float b[3][2][4];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i = 3 * q4 + k;
    float w[5][5];
#pragma unroll
    for (int u1 = 0; u1 < 5; ++u1) {
      const float4* wp = reinterpret_cast<const float4*>(s.Kp + ((i * 6 + c) * 5 + u1) * 8);
      const float4 w0 = wp[0], w1 = wp[1];
      w[u1][0] = w0.x; w[u1][1] = w0.y; w[u1][2] = w0.z; w[u1][3] = w0.w; w[u1][4] = w1.x;
    }
#pragma unroll
    for (int orow = 0; orow < 2; ++orow)
#pragma unroll
      for (int o = 0; o < 4; ++o) b[k][orow][o] = 0.0f;
    // padded rows R = p0 + rr, rr = 5..0: output row orow uses tap row u1 = orow + 4 - rr (ascending)
#pragma unroll
    for (int rr = 5; rr >= 0; --rr) {
      const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, p0 + rr, 4 * qq));
      const float4 d0 = dp[0], d1 = dp[1];
      const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
      for (int orow = 0; orow < 2; ++orow) {
        const int u1 = orow + 4 - rr;
        if (u1 < 0 || u1 > 4) continue;
        if constexpr (EXACT) {
          float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int u2 = 0; u2 < 5; ++u2)
#pragma unroll
            for (int o = 0; o < 4; ++o) rs[o] = mac<true>(rs[o], w[u1][u2], d[o - u2 + 4]);
#pragma unroll
          for (int o = 0; o < 4; ++o) b[k][orow][o] = fadd(b[k][orow][o], rs[o]);
        } else {
#pragma unroll
          for (int u2 = 0; u2 < 5; ++u2)
#pragma unroll
            for (int o = 0; o < 4; ++o) b[k][orow][o] = __fmaf_rn(w[u1][u2], d[o - u2 + 4], b[k][orow][o]);
        }
      }
    }
  }
  float acc[2][4];
  if constexpr (EXACT) {
    const int lead = (threadIdx.x & 31) & ~3;
#pragma unroll
    for (int orow = 0; orow < 2; ++orow)
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        float a = 0.0f;
#pragma unroll
        for (int src = 0; src < 4; ++src)
#pragma unroll
          for (int k = 0; k < 3; ++k) a = fadd(a, __shfl_sync(0xffffffffu, b[k][orow][o], lead + src));
        acc[orow][o] = a;
      }
  } else {
#pragma unroll
    for (int orow = 0; orow < 2; ++orow)
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        float a = (b[0][orow][o] + b[1][orow][o]) + b[2][orow][o];
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        acc[orow][o] = a;
      }
  }
  if (valid && q4 == 0) {
    // backavgpool (x0.25) + backsigmoid through c1 for the 4x8 block of c1 this quad owns
#pragma unroll
    for (int orow = 0; orow < 2; ++orow)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        float4* cp = reinterpret_cast<float4*>(s.c1 + c1_at(c, 2 * (p0 + orow) + dy, 8 * qq));
        const float4 v0 = cp[0], v1 = cp[1];
        float cv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const float dc = fmul(acc[orow][x >> 1], 0.25f);
          cv[x] = fmul(fmul(dc, cv[x]), fsub(1.0f, cv[x]));
        }
        cp[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
        cp[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
      }
  }
}

// Fast g_k2/g_b2: lane quads per (i, c) hold all 25 outputs; lane q of the quad takes rows y = 2q, 2q+1
// and the quad combines with a fixed xor tree (each s1 row feeds 5 outputs x 8 taps from registers).
template <bool ACCUM>
__device__ __forceinline__ void gk2_fast(const Smem& s, float* row, int t) {
  const int item = t >> 2, q4 = t & 3, i = item / 6, c = item - i * 6;
  float acc[5][5];
#pragma unroll
  for (int u = 0; u < 5; ++u)
#pragma unroll
    for (int v = 0; v < 5; ++v) acc[u][v] = 0.0f;
  float bsum = 0.0f;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy) {
    const int y = 2 * q4 + dy;
    const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, y + 4, 4));
    const float4 d0 = dp[0], d1 = dp[1];
    const float dr[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    bsum += ((dr[0] + dr[1]) + (dr[2] + dr[3])) + ((dr[4] + dr[5]) + (dr[6] + dr[7]));
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const float4* sp = reinterpret_cast<const float4*>(s.s1 + (c * 12 + u + y) * 12);
      const float4 a = sp[0], b = sp[1], cc = sp[2];
      const float sr[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[u][v] = __fmaf_rn(sr[v + x], dr[x], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 5; ++u)
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      float a = acc[u][v];
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      acc[u][v] = a;
    }
  bsum += __shfl_xor_sync(0xffffffffu, bsum, 1);
  bsum += __shfl_xor_sync(0xffffffffu, bsum, 2);
  // spread the 25 puts over the quad's lanes (lane q writes outputs q, q+4, ...)
#pragma unroll
  for (int k = 0; k < 25; ++k)
    if ((k & 3) == q4) put<ACCUM>(s, row, kK2 + (i * 6 + c) * 25 + k, acc[k / 5][k % 5]);
  if (c == 0 && q4 == 0) put<ACCUM>(s, row, kB2 + i, bsum);
}

// Weight-stationary backin.  Lane t < 504 -> kernel i = t / 42, channel c = t % 6 and tile group
// tg = (t % 42) / 6; it keeps the 25 weights of k2[i][c] in registers and walks tiles tg, tg+7, tg+14
// (2 rows x 4 columns of d_s1[c]), streaming six padded dz2[i] rows per tile.  The six lanes of a
// tile differ only in c, so each quarter-warp reads at most two distinct rows (broadcast).  Each
// tile's per-kernel term b_i (EXACT: the reference's nested row/outer sums; fast: FFMA) goes to
// term[i][c][p][q]; backin_combine then forms acc = (((0 + b_0) + b_1) + ... + b_11) per output in
// kernel order (network.cpp:135-138).
template <bool EXACT>
__device__ __forceinline__ void backin_ws(const Smem& s) {
  const int t = threadIdx.x;
  if (t >= 504) return;
  const int i = t / 42, r = t - i * 42, sub = r / 6, c = r - sub * 6;
  float w[5][5];
#pragma unroll
  for (int u1 = 0; u1 < 5; ++u1)
#pragma unroll
    for (int u2 = 0; u2 < 5; ++u2) w[u1][u2] = s.Kp[((i * 6 + c) * 5 + u1) * 8 + u2];
  float* term = s.term + (i * 6 + c) * 144;
#pragma unroll 1
  for (int tile = sub; tile < 18; tile += 7) {
    const int pp = tile / 3, qq = tile - pp * 3, p0 = 2 * pp;
    float b[2][4];
#pragma unroll
    for (int orow = 0; orow < 2; ++orow)
#pragma unroll
      for (int o = 0; o < 4; ++o) b[orow][o] = 0.0f;
    float d[6][8];
#pragma unroll
    for (int rr = 0; rr < 6; ++rr) {  // all six rows in flight before the first multiply
      const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, p0 + rr, 4 * qq));
      const float4 d0 = dp[0], d1 = dp[1];
      d[rr][0] = d0.x; d[rr][1] = d0.y; d[rr][2] = d0.z; d[rr][3] = d0.w;
      d[rr][4] = d1.x; d[rr][5] = d1.y; d[rr][6] = d1.z; d[rr][7] = d1.w;
    }
    // padded rows R = p0 + rr: output row orow uses tap row u1 = orow + 4 - rr, ascending as rr falls
#pragma unroll
    for (int rr = 5; rr >= 0; --rr) {
#pragma unroll
      for (int orow = 0; orow < 2; ++orow) {
        const int u1 = orow + 4 - rr;
        if (u1 < 0 || u1 > 4) continue;
        float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int u2 = 0; u2 < 5; ++u2)
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            if constexpr (EXACT) rs[o] = mac<true>(rs[o], w[u1][u2], d[rr][o - u2 + 4]);
            else b[orow][o] = __fmaf_rn(w[u1][u2], d[rr][o - u2 + 4], b[orow][o]);
          }
        if constexpr (EXACT) {
#pragma unroll
          for (int o = 0; o < 4; ++o) b[orow][o] = fadd(b[orow][o], rs[o]);
        }
      }
    }
#pragma unroll
    for (int orow = 0; orow < 2; ++orow)
      *reinterpret_cast<float4*>(term + (p0 + orow) * 12 + 4 * qq) =
          make_float4(b[orow][0], b[orow][1], b[orow][2], b[orow][3]);
  }
}

// d_s1[c][p][4qq..4qq+3] = ordered sum of the twelve kernel terms, then backavgpool + backsigmoid
// through c1 -> dz1 for the 2x8 block of c1 it feeds.  216 lanes (c, p, qq).
__device__ __forceinline__ void backin_combine(const Smem& s, int it) {
  const int c = it / 36, r = it - c * 36, p = r / 3, qq = r - p * 3;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const float4 v = *reinterpret_cast<const float4*>(s.term + (i * 6 + c) * 144 + p * 12 + 4 * qq);
    acc[0] = fadd(acc[0], v.x);
    acc[1] = fadd(acc[1], v.y);
    acc[2] = fadd(acc[2], v.z);
    acc[3] = fadd(acc[3], v.w);
  }
#pragma unroll
  for (int dy = 0; dy < 2; ++dy) {
    float4* cp = reinterpret_cast<float4*>(s.c1 + c1_at(c, 2 * p + dy, 8 * qq));
    const float4 v0 = cp[0], v1 = cp[1];
    float cv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const float dc = fmul(acc[x >> 1], 0.25f);
      cv[x] = fmul(fmul(dc, cv[x]), fsub(1.0f, cv[x]));
    }
    cp[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
    cp[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
  }
}

template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void stage_conv1_back(const Smem& s, const float* img, float* row) {
  const float* dz1 = s.c1;
  if constexpr (EXACT) {
#if TLB_C1BACK_EXACT_BLOCKED
    stage_conv1_back_exact_blocked<ACCUM>(s, img, row);
#else
    for (int it = threadIdx.x; it < 156; it += blockDim.x) stage_conv1_back_lane_exact<ACCUM>(s, row, it);
#endif
  } else {
    const int it = threadIdx.x;
    if (it < 144) {  // (i, y): 25 row-partials + the bias row-partial
      const int i = it / 24, y = it - i * 24;
      const float4* dp = reinterpret_cast<const float4*>(dz1 + c1_at(i, y, 0));
      float dr[24];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float4 t = dp[q];
        dr[4 * q] = t.x; dr[4 * q + 1] = t.y; dr[4 * q + 2] = t.z; dr[4 * q + 3] = t.w;
      }
      float bias = 0.0f;
#pragma unroll
      for (int x = 0; x < 24; ++x) bias += dr[x];
      float* out = s.red + it * 26;
      out[25] = bias;
#pragma unroll 1
      for (int u = 0; u < 5; ++u) {
        const float4* ip = reinterpret_cast<const float4*>(img + (u + y) * 28);
        float ir[28];
#pragma unroll
        for (int q = 0; q < 7; ++q) {
          const float4 t = ip[q];
          ir[4 * q] = t.x; ir[4 * q + 1] = t.y; ir[4 * q + 2] = t.z; ir[4 * q + 3] = t.w;
        }
        float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int x = 0; x < 24; ++x)
#pragma unroll
          for (int v = 0; v < 5; ++v) acc[v] = __fmaf_rn(ir[x + v], dr[x], acc[v]);
#pragma unroll
        for (int v = 0; v < 5; ++v) out[u * 5 + v] = acc[v];
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 156; t += blockDim.x) {
      float acc = 0.0f;
      if (t < 150) {
        const int i = t / 25, k = t - i * 25;
#pragma unroll 8
        for (int y = 0; y < 24; ++y) acc += s.red[(i * 24 + y) * 26 + k];
        put<ACCUM>(s, row, kK1 + t, acc);
      } else {
        const int i = t - 150;
#pragma unroll 8
        for (int y = 0; y < 24; ++y) acc += s.red[(i * 24 + y) * 26 + 25];
        put<ACCUM>(s, row, kB1 + i, acc);
      }
    }
  }
}

template <bool EXACT, bool ACCUM, int GLO = 0, bool ROWS = false>
__device__ __forceinline__ void stage_conv1_back_gk2_legacy(const Smem& s, const float* img, float* row) {
  constexpr int kGk2 = EXACT ? 372 : ROWS ? 360 : 288;
  const int t = threadIdx.x;
  if constexpr (!EXACT && TLB_C1BACK_GROUP2) {
    if (blockDim.x >= 512) {  // C1 gradient on warps 0-8, the remaining g_k2 lanes on warps 9+
      if (t < 288) {
        conv1_back_fast_group2<ACCUM>(s, img, row);
      } else {
        for (int item = GLO + t - 288; item < kGk2; item += blockDim.x - 288) {
          if constexpr (ROWS) gk2_rows<ACCUM>(s, row, item);
          else gk2_fast<ACCUM>(s, row, item);
        }
      }
      return;
    }
  }
  static_assert(!ROWS || !EXACT, "row-form g_k2 is a fast-mode stage");
  if constexpr (EXACT && GLO > 0) {  // V15: ordered C1 chains on the first warps, g_k2 chains after them
    constexpr int kC1 = TLB_V15_C1_LANES ? 160 : 96;  // one chain per lane (5 warps) | blocked (3 warps)
    if (t < kC1) {
      if constexpr (TLB_V15_C1_LANES) {
        if (t < 156) stage_conv1_back_lane_exact<ACCUM>(s, row, t);
      } else {
        stage_conv1_back_exact_blocked<ACCUM>(s, img, row);
      }
    } else {
      for (int item = GLO + t - kC1; item < kGk2; item += blockDim.x - kC1) gk2_exact<ACCUM>(s, row, item);
    }
    return;
  }
  if (t < 160) {
    if constexpr (EXACT) {
      if (t < 156) stage_conv1_back_lane_exact<ACCUM>(s, row, t);
    } else {
      conv1_back_fast_group<ACCUM>(s, img, row);
    }
  } else {
    for (int item = GLO + t - 160; item < kGk2; item += blockDim.x - 160) {
      if constexpr (EXACT) gk2_exact<ACCUM>(s, row, item);
      else if constexpr (ROWS) gk2_rows<ACCUM>(s, row, item);
      else gk2_fast<ACCUM>(s, row, item);
    }
  }
}

// C2 backward stage.  V = 0: backin lane quads on warps 0-13 (432 lanes), then the g_k2/g_b2 lanes;
// V = 1: one backin lane per item on warps 0-3, concurrent with the g_k2/g_b2 lanes on warps 4+.
template <bool EXACT, bool ACCUM, int V>
__device__ __forceinline__ void stage_conv2_back_legacy(const Smem& s, float* row) {
  constexpr int kGk2 = EXACT ? 372 : 288;  // exact: 360 (i,c,u) lanes + 12 g_b2; fast: 72 quads
  if constexpr (V == 0) {
    constexpr int kBackin = 448;  // 108 quads = 432 lanes, padded to 14 warps
    for (int it = threadIdx.x; it < kBackin + kGk2; it += blockDim.x) {
      if (it < kBackin) {
        backin_quad<EXACT>(s, it, it < 432);
      } else if constexpr (EXACT) {
        gk2_exact<ACCUM>(s, row, it - kBackin);
      } else {
        gk2_fast<ACCUM>(s, row, it - kBackin);
      }
    }
  } else if constexpr (V == 1) {
    constexpr int kBackin = 128;  // 108 items, padded to 4 whole warps
    for (int it = threadIdx.x; it < kBackin + kGk2; it += blockDim.x) {
      if (it < kBackin) {
        if (it < 108) backin_item<EXACT>(s, it);
      } else if constexpr (EXACT) {
        gk2_exact<ACCUM>(s, row, it - kBackin);
      } else {
        gk2_fast<ACCUM>(s, row, it - kBackin);
      }
    }
  } else if constexpr (V == 6 || V == 7 || V == 8) {
    // V = 6/7/8 (fast only): scatter-form backin rows with 2 / 4 / 4 kernel splits per (c, p) beside
    // the g_k2/g_b2 lane quads (8: weights from P)
    static_assert(!EXACT, "scatter-form backin reorders the reference's sums");
    constexpr int kSplits = V == 6 ? 2 : 4;
    constexpr int kBackin = (72 * kSplits + 31) / 32 * 32;
    for (int it = threadIdx.x; it < kBackin + kGk2; it += blockDim.x) {
      if (it < kBackin) {
        backin_rows<kSplits, V == 8>(s, it);
      } else {
        gk2_fast<ACCUM>(s, row, it - kBackin);
      }
    }
  } else if constexpr (V == 9) {
    // V = 9 (fast only): scatter-form backin rows (4 splits, weights from P) alone on warps 0-8;
    // g_k2/g_b2 runs beside the C1 gradient
    static_assert(!EXACT, "scatter-form backin reorders the reference's sums");
    for (int it = threadIdx.x; it < 288; it += blockDim.x) backin_rows<4, true>(s, it);
  } else if constexpr (V == 15) {
    // V = 15 (EXACT): scatter-form exact backin on warps 0-8 beside ordered g_k2 chains 0-223 on warps
    // 9-15; chains 224-371 run beside the C1 gradient
    static_assert(EXACT, "V15 is the EXACT schedule");
    for (int it = threadIdx.x; it < 288 + gk2_split_lanes(15); it += blockDim.x) {
      if (it < 288) backin_rows_exact(s, it);
      else gk2_exact<ACCUM>(s, row, it - 288);
    }
  } else if constexpr (V == 14) {
    // V = 14 (fast only): backin rows on warps 0-8 beside g_k2 row lanes 0-223 on warps 9-15; row
    // lanes 224-359 run beside the C1 gradient
    static_assert(!EXACT, "scatter-form backin reorders the reference's sums");
    for (int it = threadIdx.x; it < 288 + gk2_split_lanes(14); it += blockDim.x) {
      if (it < 288) backin_rows<4, true>(s, it);
      else gk2_rows<ACCUM>(s, row, it - 288);
    }
  } else if constexpr (V >= 10 && V <= 13) {
    // V = 10..13 (fast only): backin rows on warps 0-8 beside the first gk2_split_lanes(V) g_k2 quad
    // lanes on warps 9-15; the remaining quads run beside the C1 gradient
    static_assert(!EXACT, "scatter-form backin reorders the reference's sums");
    for (int it = threadIdx.x; it < 288 + gk2_split_lanes(V); it += blockDim.x) {  // whole warps per round
      if (it < 288) backin_rows<4, true>(s, it);
      else gk2_fast<ACCUM>(s, row, it - 288);
    }
  } else if constexpr (V == 4) {
    // V = 4: backin only, one lane per item on warps 0-3 (g_k2 runs later, beside the C1 gradient)
    if (threadIdx.x < 108) backin_item<EXACT>(s, threadIdx.x);
  } else if constexpr (V == 5) {
    // V = 5: backin only, lane quads over 14 warps (g_k2 runs later, beside the C1 gradient)
    for (int it = threadIdx.x; it < 448; it += blockDim.x) backin_quad<EXACT>(s, it, it < 432);
  } else if constexpr (V == 3) {
    // V = 3: weight-stationary backin over all lanes, then the ordered kernel combine (224 lanes)
    // beside the g_k2/g_b2 lanes.
    backin_ws<EXACT>(s);
    __syncthreads();
    constexpr int kComb = 224;  // 216 (c, p, qq) lanes padded to 7 warps
    for (int it = threadIdx.x; it < kComb + kGk2; it += blockDim.x) {
      if (it < kComb) {
        if (it < 216) backin_combine(s, it);
      } else if constexpr (EXACT) {
        gk2_exact<ACCUM>(s, row, it - kComb);
      } else {
        gk2_fast<ACCUM>(s, row, it - kComb);
      }
    }
  } else {
    // V = 2: lane pairs per backin item (224 lanes = 7 warps) beside the g_k2/g_b2 lanes
    constexpr int kBackin = 224;
    for (int it = threadIdx.x; it < kBackin + kGk2; it += blockDim.x) {
      if (it < kBackin) {
        backin_tile<EXACT, 2>(s, it, it < 216);
      } else if constexpr (EXACT) {
        gk2_exact<ACCUM>(s, row, it - kBackin);
      } else {
        gk2_fast<ACCUM>(s, row, it - kBackin);
      }
    }
  }
}

}  // namespace tlb
