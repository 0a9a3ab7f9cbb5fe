// objective.cu -- rows a6 + a8: K5 (per-configuration tier counts from the cumulative
// stack tables, closed forms of DESIGN.md "Stack path") fused with K7 (the fp64 fluid
// objective model of Eq. 1 / Eq. 2, R25-R33).
//
// THIS TRANSLATION UNIT IS COMPILED WITH -fmad=false: every floating-point operation is
// performed as written (IEEE +, -, *, / correctly rounded, no contraction, no libm), in
// the fixed order of DESIGN.md section 3, so the results are bit-identical to the oracle.
#include "eval.cuh"

namespace kareto {

__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double gb(uint64_t c, uint64_t Bb) { return (double)(c * Bb) / 1e9; }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ double phi_iops(const kareto_model &m, double u) {  // R32, right-continuous
  double v = 0.0;
  for (int i = 0; i < m.n_phi; i++) {
    if (u >= m.phi[i].breakpoint) {
      double top = (i + 1 < m.n_phi) ? dmin(u, m.phi[i + 1].breakpoint) : u;
      v = (v + m.phi[i].jump) + m.phi[i].rate * (top - m.phi[i].breakpoint);
    }
  }
  return v;
}

__global__ void k_objective(StackTables T, const kareto_config *__restrict__ cfg, const CfgDev *__restrict__ cd,
                            const uint32_t *__restrict__ tix, const uint32_t *__restrict__ ttl_ms, int64_t n,
                            kareto_model m, ModelConsts mc, const kareto_counts *__restrict__ given,
                            kareto_counts *__restrict__ counts, double *__restrict__ obj) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const kareto_config c = cfg[i];
    const bool ttl = c.cap[2] == KARETO_INF;
    const uint64_t c1 = c.cap[0];
    kareto_counts k;
    if (given) {  // counts from the K6 replay: objective only
      k = given[i];
    } else {
    const CfgDev x = cd[i];
    const int any = T.ntc;
    const unsigned long long *Ca = T.C1 + (size_t)any * T.nb, *Sa = T.S1 + (size_t)any * T.nb;
    const uint64_t N = mc.N, U = mc.U;
    const uint64_t c12 = c1 + c.cap[1];
    uint64_t h1 = Ca[x.i1], h12 = Ca[x.i12];
    k.hit[0] = h1;
    k.hit[1] = h12 - h1;
    uint64_t hps = Sa[x.i12];
    k.evict[0] = (N - T.CD[x.i1]) - umin64(c1, U);
    k.evict[1] = (N - T.CD[x.i12]) - umin64(c12, U);
    k.bytetime_block_ms = 0;
    k.resident_after_hole = 0;
    if (!ttl) {
      const unsigned long long *Ct = T.C1 + (size_t)x.tc * T.nb, *St = T.S1 + (size_t)x.tc * T.nb;
      k.hit[2] = Ct[x.iC] - Ct[x.i12];
      hps += St[x.iC] - St[x.i12];
      uint64_t C = c12 + c.cap[2];
      k.evict[2] = (x.tc == T.ntc) ? (N - T.CD[x.iC]) - umin64(C, U) : KARETO_NA;
      k.disk_writes = c.cap[2] > 0 ? k.evict[1] : 0;
    } else {
      uint64_t h3 = 0, w = 0, bt = 0;
      const int G = T.G, nt1 = T.ntt + 1;
      for (int g = 0; g < G; g++) {
        uint32_t t = tix[(size_t)x.row * G + g];
        uint64_t tau = ttl_ms[(size_t)x.row * G + g];
        size_t all = ((size_t)T.nb12 * G + g) * nt1 + t;
        size_t in = ((size_t)x.i12t * G + g) * nt1 + t;
        uint64_t ndel = T.C2[all];
        h3 += ndel - T.C2[in];
        hps += T.S2[all] - T.S2[in];
        uint64_t late = T.Rg[g] - ndel;
        w += T.Ug[g] + late;
        bt += T.Ug[g] * tau + T.SDg[(size_t)g * nt1 + t] + tau * late;
      }
      k.hit[2] = h3;
      k.disk_writes = w;
      k.bytetime_block_ms = bt;
      k.evict[2] = 0;
    }
    k.hit_pos_sum = hps;
    k.miss = N - k.hit[0] - k.hit[1] - k.hit[2];
    }
    if (counts) counts[i] = k;

    // ---- K7: fluid objective, DESIGN.md section 3 (fixed order, no FMA)
    const uint64_t Bb = m.block_bytes;
    const uint64_t Hc = k.hit[0] + k.hit[1] + k.hit[2];
    const uint64_t S = 16 * m.alpha_ps * Hc + m.beta_ps * (256 * k.hit_pos_sum + 120 * Hc);
    const double prefill_s = (double)(mc.P0 - S) * 1e-12;
    const double decode_s = (double)(m.dec_ps * mc.O) * 1e-12;
    const kareto_medium md = m.media[c.medium];
    const double prov_gb = ttl ? m.ttl_prov_gb : gb(c.cap[2], Bb);
    const double bw_disk = dmin(md.bw_max, md.bw_base + md.bw_slope * prov_gb);
    const double dram_s = (double)(k.hit[1] * Bb) / m.bw_dram;
    const uint64_t io = k.hit[2] + k.disk_writes;
    const double disk_s = io == 0 ? 0.0 : (double)(io * Bb) / bw_disk;
    const double busy_s = (((prefill_s + decode_s) + dram_s) + disk_s) / (double)m.instances;
    const double T_s = (double)mc.span_ms * 1e-3;
    const double M_s = dmax(T_s, busy_s);
    const double f1 = 1e3 * ((((prefill_s + dram_s) + disk_s) / (double)mc.R) + dmax(0.0, busy_s - T_s) / 2.0);
    const double f2 = -((double)(mc.Ltok + mc.O) / M_s);
    const double hours = M_s / 3600.0;
    double cost = (m.c_hw * (double)((int64_t)m.instances * m.gpus_per_instance)) * hours;
    cost = cost + (m.p_hbm * gb(c1, Bb)) * hours;
    cost = cost + (m.p_dram * gb(c.cap[1], Bb)) * hours;
    if (ttl) cost = cost + (md.price * ((double)Bb / 1e9)) * ((double)k.bytetime_block_ms / 3.6e6);
    else cost = cost + (md.price * gb(c.cap[2], Bb)) * hours;
    const double iops = ((double)io * m.iops_per_block) / M_s;
    cost = cost + (phi_iops(m, iops) / 730.0) * hours;
    if (obj) {
      obj[3 * i + 0] = f1;
      obj[3 * i + 1] = f2;
      obj[3 * i + 2] = cost;
    }
  }
}

void launch_objective(kareto_ctx *ctx, const StackTables &T, const kareto_config *cfg, const CfgDev *cd,
                      const uint32_t *tix, const uint32_t *ttl_ms, int64_t n, const kareto_model *model,
                      ModelConsts mc, const kareto_counts *given, kareto_counts *counts, double *obj) {
  if (n <= 0) return;
  Pass ps(ctx, given ? "K7_objective" : "K5K7_objective", 1, 1);
  k_objective<<<grid_for(n, 128, 8 * ctx->num_sms), 128, 0, ctx->stream>>>(T, cfg, cd, tix, ttl_ms, n, *model, mc,
                                                                           given, counts, obj);
}

}  // namespace kareto
