// On-device KHI / thermal initialisation.
//
// Reference: pic/sim.py:239-302 `init_khi` -- per cell a quiet-start
// sub-lattice of ppc = px*py*pz particles at ((i+1/2)/px, (j+1/2)/py,
// (k+1/2)/pz) (x fastest, _near_cubic_factors), counter-streaming v_x =
// +-v0 split at y = ny/2, v_y = amp sin(2 pi x / Lx), u = gamma v, plus
// N(0, thermal_u^2) jitter per component.  The host path (numpy) reproduces
// the reference's default_rng stream bit for bit; this kernel is the fast
// path for 10^8-10^9 particles: identical deterministic placement and
// velocity profile, thermal jitter from a counter-based Philox generator
// keyed by (seed, species) and the particle's global index (so it is
// independent of the launch geometry and of the z-slab decomposition).
// One thread per (cell, sub-lattice site); the columns are written directly
// (frame j of cell c holds site j), fully coalesced.
#include <curand_kernel.h>

#include "common.cuh"

namespace kwb {

template <typename F>
__global__ void init_khi_kernel(Geo g, kwb_init ini, StoreT<F> st) {
    const int V = g.scx * g.scy * g.scz, K = st.frames, ppc = ini.ppc;
    const int64_t ncol = (int64_t)g.gx * g.gy * g.gz * V;
    const int64_t total = ncol * ppc;
    const double two_pi = 6.283185307179586;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / ncol);           // site (frame) index: frame-major, coalesced
        const int64_t colx = idx - (int64_t)j * ncol;
        const int s = (int)(colx / V), c = (int)(colx % V);
        const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
        const int cx = bx * g.scx + c % g.scx, cy = by * g.scy + (c / g.scx) % g.scy,
                  cz = bz * g.scz + c / (g.scx * g.scy);
        const int ix = j % ini.px, iy = (j / ini.px) % ini.py, iz = j / (ini.px * ini.py);
        const double ox = (ix + 0.5) / ini.px, oy = (iy + 0.5) / ini.py, oz = (iz + 0.5) / ini.pz;
        const int gy = cy + ini.y_offset;           // global cell for the KHI profile
        const double vx = gy < ini.global_ny / 2 ? ini.stream_velocity : -ini.stream_velocity;
        const double xa = ((double)(cx + ini.x_offset) + ox) * g.dx;
        const double vy = ini.perturbation * sin(two_pi * xa / (ini.global_nx * g.dx));
        const double gam = 1.0 / sqrt(1.0 - (vx * vx + vy * vy));
        double ux = vx * gam, uy = vy * gam, uz = 0.0;
        if (ini.thermal_u > 0.0) {
            // global particle id: (global cell, site) -> independent of slabs/launch
            const int64_t gz = cz + ini.z_offset;
            const int64_t gcell = (gz * ini.global_ny + gy) * ini.global_nx + (cx + ini.x_offset);
            curandStatePhilox4_32_10_t rs;
            curand_init(ini.seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(ini.species_index + 1)),
                        (unsigned long long)(gcell * ppc + j), 0, &rs);
            const double2 n01 = curand_normal2_double(&rs);
            const double2 n23 = curand_normal2_double(&rs);
            ux += ini.thermal_u * n01.x;
            uy += ini.thermal_u * n01.y;
            uz += ini.thermal_u * n23.x;
        }
        const int64_t q = ((int64_t)s * K + j) * V + c;
        st.ox[q] = (F)ox; st.oy[q] = (F)oy; st.oz[q] = (F)oz;
        st.ux[q] = (F)ux; st.uy[q] = (F)uy; st.uz[q] = (F)uz;
        st.w[q] = (F)ini.weight;
        if (j == 0) { st.front[colx] = ppc; st.back[colx] = 0; }
    }
}

}  // namespace kwb

using namespace kwb;

extern "C" int kwb_init_khi(const kwb_grid *g, const kwb_init *ini, const kwb_store *st,
                            kwb_stream_t stream) {
    if (!g || !ini || !st || !st->ox || !st->front || !st->back) {
        kwb_set_error("init_khi: NULL argument");
        return KWB_EINVAL;
    }
    if (ini->ppc <= 0 || ini->px * ini->py * ini->pz != ini->ppc) {
        kwb_set_error("init_khi: ppc must equal px*py*pz");
        return KWB_EINVAL;
    }
    if (st->frames_per_sc < ini->ppc) {
        kwb_set_error("init_khi: %d frames per super cell < %d particles per cell",
                      st->frames_per_sc, ini->ppc);
        return KWB_EINVAL;
    }
    if (g->dtype != KWB_F32 && g->dtype != KWB_F64) {
        kwb_set_error("init_khi: bad dtype");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 16;
    if (g->dtype == KWB_F32)
        init_khi_kernel<float><<<blocks, 256, 0, s>>>(geo, *ini, store_of<float>(*st));
    else
        init_khi_kernel<double><<<blocks, 256, 0, s>>>(geo, *ini, store_of<double>(*st));
    return kwb_check_launch("init_khi_kernel");
}

unsigned long long kwb_chk_read_init(int reset) {
#ifdef KWB_CHECKS
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, kwb::kwb_chk_count, sizeof(v));
    if (reset) {
        const unsigned long long z = 0;
        cudaMemcpyToSymbol(kwb::kwb_chk_count, &z, sizeof(z));
    }
    return v;
#else
    (void)reset;
    return 0;
#endif
}
