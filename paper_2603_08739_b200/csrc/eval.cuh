// eval.cuh -- internals shared by eval.cu (K4 histograms, sharding, collectives) and
// objective.cu (K5+K7 fused counts + fp64 objective, compiled with -fmad=false).
#pragma once
#include "internal.cuh"

namespace kareto {

// Cumulative tables produced by K4 for one evaluation (device pointers).
struct StackTables {
  // boundary values (clamped to U), sorted unique
  const uint64_t *Bd;  int nb;     // all c1 / c12 / C boundaries
  const uint32_t *Tc;  int ntc;    // finite uniform CAPACITY TTLs
  // C1[tc][i] / S1[tc][i]: #{reuse access: d <= Bd[i], delta <= Tc[tc]} and sum k over them,
  // tc == ntc: any delta.  Layout [(ntc+1)][nb]
  const unsigned long long *C1, *S1;
  // CD[i] = #{reuse access: D <= Bd[i]}
  const unsigned long long *CD;
  // TTL mode (may be empty)
  const uint64_t *B12; int nb12;   // c12 boundaries of TTL configurations
  const uint32_t *Tt;  int ntt;    // finite TTL values of the rows used by TTL configurations
  int G;                           // groups K+1
  // C2[(i*G + g)*(ntt+1) + t]: #{reuse: d <= B12[i] (i == nb12: any d), group g, delta <= Tt[t]
  // (t == ntt: any)}; S2 the sum of k over them.  i ranges over [0, nb12]
  const unsigned long long *C2, *S2;
  // per group delta sums: SDg[g*(ntt+1) + t] = sum of delta over reuse accesses of group g with
  // delta <= Tt[t]
  const unsigned long long *SDg;
  const unsigned long long *Ug, *Rg;  // [G] unique blocks / reuse events per group
};

struct ModelConsts {  // trace + model constants for the objective (host-computed integers)
  uint64_t P0;          // sum_r alpha L_r + beta L_r (L_r - 1) / 2   (ps)
  uint64_t R, N, U, Ltok, O;
  int64_t span_ms;
};

struct CfgDev {       // per-configuration lookup indices (host-computed)
  int32_t i1, i12, iC;   // indices into Bd of clamp(c1), clamp(c12), clamp(C) (iC = -1: TTL mode)
  int32_t tc;            // CAPACITY uniform-TTL column (ntc = infinite)
  int32_t i12t;          // TTL mode: index into B12
  int32_t row;           // TTL mode: tuner row
};

// K5 + K7: counts from the cumulative tables, then the fp64 objective (objective.cu)
void launch_objective(kareto_ctx *ctx, const StackTables &T, const kareto_config *cfg, const CfgDev *cd,
                      const uint32_t *ttl_t_index /*[n_rows][G] index into Tt*/, const uint32_t *ttl_ms,
                      int64_t n, const kareto_model *model, ModelConsts mc, const kareto_counts *given,
                      kareto_counts *counts, double *obj);

}  // namespace kareto
