// prepass.cuh -- layout of the per-step surfel prepass (ss_surfel_prepass):
// the view-independent per-surfel state one optimisation step's views share.
// Caller-owned buffer of ss_surfel_prepass_bytes(n): PreGeom[n], PreShade[n],
// PreDiff[n].
#pragma once
#include <cstdint>

// float32 scaled tangent frame (the preprocess kernel's operations, bit-identical)
struct PreGeom {
    float su0, su1, su2, sv0;
    float sv1, sv2;
    int finite, zero_norm;
};
// float64 shading inputs and the diffuse lookup of the forward (shading.py:463-471)
struct PreShade {
    double n[3], l_d[3];
    float alb[3], m, r;
    uint32_t cell;   // diffuse cell i0 | j0 << 16
    uint32_t dv_ok;  // diffuse dv_ok
    uint32_t pad;
};
// The float32 diffuse state of the chain kernel's shading adjoint (normal-only,
// so once per step): the lookup value and texel derivatives on the float64
// forward's cell, the linear map of coord_grad_to_dir(n) (shading.py:182-197):
// dL/dn = (gfu a0, gfu a1, gfv b2), and the bilinear fractions of the cell.
struct PreDiff {
    float l_d[3], gu[3], gv[3];
    float a0, a1, b2;
    float tu, tv;
    float pad[2];
};
static_assert(sizeof(PreGeom) == 32 && sizeof(PreShade) == 80 && sizeof(PreDiff) == 64, "prepass layout");

__host__ __device__ inline const PreShade *prepass_shade(const void *p, int n) {
    return reinterpret_cast<const PreShade *>(reinterpret_cast<const PreGeom *>(p) + n);
}
__host__ __device__ inline const PreDiff *prepass_diff(const void *p, int n) {
    return reinterpret_cast<const PreDiff *>(prepass_shade(p, n) + n);
}
