// Certified FP32 projection of grid voxel centres (shared by the carve and
// the exact-isovalue kernel): see the derivation below.
#pragma once
#include "fvv_common.cuh"

namespace fvv {

// ---- FP32 pre-classification --------------------------------------------
// Without distortion, u = U/Z and v = V/Z with (U, V, Z) affine in the voxel
// indices (i, j, k): U = U0 + i Ui + j Uj + k Uk (K [R|t] applied to the
// voxel centre). Each (voxel, camera) test is first evaluated in FP32 from
// these per-(grid, camera) coefficients together with a rigorous bound E on
// |u32 - u| (and on v, Z). When u32 (v32) is farther than E from every
// half-integer, rint(u) of the reference's float64 chain equals rintf(u32),
// so the test's outcome (frustum, silhouette bit) is decided exactly in
// FP32. Otherwise the camera is "ambiguous"; a voxel with an ambiguous
// camera and no camera that rejects it is re-run through the float64 chain.
// Bound: with eps = 2^-24 and S = |U0| + i|Ui| + j|Uj| + k|Uk| (bounded by
// its value at the far grid corner), coefficient rounding plus the three
// fmaf roundings give |U32 - U| <= 4 eps S_U (same for Z); then
// |U32/Z32 - U/Z| <= 4 eps (S_U + |u| S_Z) / Z32 to first order, plus
// 3 eps |u| for the reciprocal (MUFU.RCP refined by one Newton step: within
// ~1 ulp) and the product; the float64 chain's own error (< 1e-9 px at these
// magnitudes) is covered by an absolute 2^-20; the whole bound is scaled by
// 1.25 for second-order terms and the rounding of E itself (and the
// per-camera constants
// inflated by 1%). The sign of Z is certain once |Z32| > ez; when every
// voxel of the grid has Z beyond that (Z is affine, its minimum is at a
// grid corner) the sign checks are skipped. A |u32| beyond ulim lies outside
// the image whatever its rounding. Cameras with lens distortion always take
// the float64 chain (ez = inf).
struct __align__(16) CamAffine {
  float u[4], v[4], z[4];  // constant, i, j, k coefficients
  float su, sv, sz, ez;    // magnitude sums at the far corner; |Z32 - Z| bound
  float zsafe, ulim, bu, bv;  // E_u = (|u|+1)(A rz + C) + bu rz + 2^-20
  float A;                 // 8 eps sz
  int w, h;
  int sil_off;             // word offset of the camera's silhouette plane (carve_affine)
  int sil_stride;          // its words per row
  int pad[3];
};

constexpr float kEps = 5.9604645e-8f;  // 2^-24

__device__ __forceinline__ void cam_affine(const fvv_camera &c, const fvv_grid &g, CamAffine &a) {
  const double hs = 0.5 * g.spacing;
  const double ox = g.origin[0] + hs, oy = g.origin[1] + hs, oz = g.origin[2] + hs;
  // rows of K [R|t] (no distortion): U = fx X + fx skew Y + cx Z, V = fy Y + cy Z
  double ku[4], kv[4], kz[4];
  for (int m = 0; m < 3; ++m) {
    const double rx = c.R[m], ry = c.R[3 + m], rz = c.R[6 + m];  // column m of R
    ku[1 + m] = g.spacing * (c.fx * rx + c.fx * c.skew * ry + c.cx * rz);
    kv[1 + m] = g.spacing * (c.fy * ry + c.cy * rz);
    kz[1 + m] = g.spacing * rz;
  }
  const double X = c.R[0] * ox + c.R[1] * oy + c.R[2] * oz + c.t[0];
  const double Y = c.R[3] * ox + c.R[4] * oy + c.R[5] * oz + c.t[1];
  const double Z = c.R[6] * ox + c.R[7] * oy + c.R[8] * oz + c.t[2];
  ku[0] = c.fx * X + c.fx * c.skew * Y + c.cx * Z;
  kv[0] = c.fy * Y + c.cy * Z;
  kz[0] = Z;
  const double n[3] = {(double)(g.dims[0] - 1), (double)(g.dims[1] - 1), (double)(g.dims[2] - 1)};
  double su = fabs(ku[0]), sv = fabs(kv[0]), sz = fabs(kz[0]), zmin = kz[0];
  for (int m = 0; m < 3; ++m) {
    su += n[m] * fabs(ku[1 + m]);
    sv += n[m] * fabs(kv[1 + m]);
    sz += n[m] * fabs(kz[1 + m]);
    zmin += fmin(0.0, n[m] * kz[1 + m]);
  }
  for (int m = 0; m < 4; ++m) {
    a.u[m] = (float)ku[m];
    a.v[m] = (float)kv[m];
    a.z[m] = (float)kz[m];
  }
  // the double-side sums above carry ~1e-16 relative error; inflate slightly
  su *= 1.0001;
  sv *= 1.0001;
  sz *= 1.0001;
  a.su = (float)su;
  a.sv = (float)sv;
  a.sz = (float)sz;
  const double e4 = 4.0 * (double)kEps;
  const double ez = 2.0 * e4 * sz + 1e-6;
  a.ez = c.has_distortion ? INFINITY : (float)ez;
  a.w = c.width;
  a.h = c.height;
  const double ulim = (double)(c.width > c.height ? c.width : c.height) + 2.0;
  a.ulim = (float)ulim;
  // every voxel has Z >= zmin, so Z32 >= zmin - ez; below zsafe the per-test
  // sign checks run first
  const double zsafe = (zmin - 2.0 * ez) * (1.0 - 1e-6);
  a.zsafe = (!c.has_distortion && zsafe > ez) ? (float)zsafe : INFINITY;
  a.A = (float)(5.0 * (double)kEps * sz * 1.01);  // 1.25 * 4 eps
  a.bu = (float)(5.0 * (double)kEps * su * 1.01);
  a.bv = (float)(5.0 * (double)kEps * sv * 1.01);
}

enum : int { kOut = 0, kIn = 1, kAmb = 2 };

// 1/z to ~1 ulp: MUFU.RCP (<= 2 ulp) refined by one Newton step. Callers
// pass z >= ez >= 1e-6 (or 1): a normal float, so the flush-to-zero
// approximation is the plain one without __fdividef's range handling.
__device__ __forceinline__ float recip(float z) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(z));
  return fmaf(r, fmaf(-z, r, 1.0f), r);
}

// FP32 classification of one (voxel, camera): kOut (not in frustum), kIn
// (in frustum at pixel (px, py)), kAmb (undecided in FP32).
__device__ __forceinline__ int classify32(const CamAffine &a, float fi, float fj, float fk,
                                          int &px, int &py) {
  const float Z = fmaf(fk, a.z[3], fmaf(fj, a.z[2], fmaf(fi, a.z[1], a.z[0])));
  const float U = fmaf(fk, a.u[3], fmaf(fj, a.u[2], fmaf(fi, a.u[1], a.u[0])));
  const float V = fmaf(fk, a.v[3], fmaf(fj, a.v[2], fmaf(fi, a.v[1], a.v[0])));
  // E = 1.25 (4 eps (|u| S_Z + S_U) / Z + 3 eps |u|) + 2^-20, |u| -> |u32| + 1
  if (!(Z >= a.zsafe)) {
    if (Z <= -a.ez) return kOut;  // Z < 0 for certain
    if (Z < a.ez) return kAmb;
  }
  const float rz = recip(Z);
  const float k = fmaf(a.A, rz, 3.75f * kEps);
  const float eu = fmaf(fabsf(U * rz) + 1.0f, k, fmaf(a.bu, rz, 9.5367432e-7f));
  const float ev = fmaf(fabsf(V * rz) + 1.0f, k, fmaf(a.bv, rz, 9.5367432e-7f));
  const float u = U * rz, v = V * rz;
  const float ru = rintf(u), rv = rintf(v);
  px = (int)ru;
  py = (int)rv;
  const bool in = (unsigned)px < (unsigned)a.w && (unsigned)py < (unsigned)a.h;
  // beyond ulim the point is off the image whatever its rounding
  const bool amb = (fabsf(u - ru) >= 0.5f - eu && fabsf(u) <= a.ulim) ||
                   (fabsf(v - rv) >= 0.5f - ev && fabsf(v) <= a.ulim);
  return amb ? kAmb : (in ? kIn : kOut);
}

// classify32 for a voxel of a box over which the camera's Z is certainly
// positive (every box corner has Z32 >= ez; Z is affine) and whose rounding
// bounds are at most eu, ev (box_bounds below): the same decisions without
// the per-voxel sign checks and error terms.
__device__ __forceinline__ int classify32_box(const CamAffine &a, float eu, float ev, float fi,
                                              float fj, float fk, int &px, int &py) {
  const float Z = fmaf(fk, a.z[3], fmaf(fj, a.z[2], fmaf(fi, a.z[1], a.z[0])));
  const float U = fmaf(fk, a.u[3], fmaf(fj, a.u[2], fmaf(fi, a.u[1], a.u[0])));
  const float V = fmaf(fk, a.v[3], fmaf(fj, a.v[2], fmaf(fi, a.v[1], a.v[0])));
  const float rz = recip(Z);
  const float u = U * rz, v = V * rz;
  const float ru = rintf(u), rv = rintf(v);
  px = (int)ru;
  py = (int)rv;
  const bool in = (unsigned)px < (unsigned)a.w && (unsigned)py < (unsigned)a.h;
  const bool amb = (fabsf(u - ru) >= 0.5f - eu && fabsf(u) <= a.ulim) ||
                   (fabsf(v - rv) >= 0.5f - ev && fabsf(v) <= a.ulim);
  return amb ? kAmb : (in ? kIn : kOut);
}

// Rounding bounds valid for every voxel of a box from the box's corner
// values: classify32's E = (|u| + 1) k(rz) + bu rz + 2^-20 grows with |u| and
// with rz = 1/Z, and over the box |u| and rz peak at corners (u is
// linear-fractional, Z affine and positive), so the bound at (max |u|,
// max rz) covers every voxel; inflated for the rounding of this evaluation.
__device__ __forceinline__ void box_bounds(const CamAffine &a, float umax, float vmax, float rzmax,
                                           float &eu, float &ev) {
  const float k = fmaf(a.A, rzmax, 3.75f * kEps);
  eu = (fmaf(umax + 1.0f, k, fmaf(a.bu, rzmax, 9.5367432e-7f))) * 1.001f + 1e-7f;
  ev = (fmaf(vmax + 1.0f, k, fmaf(a.bv, rzmax, 9.5367432e-7f))) * 1.001f + 1e-7f;
}

}  // namespace fvv
