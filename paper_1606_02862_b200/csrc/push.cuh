// Split advance, part 1: gather -> Boris push -> move for every particle of
// a super cell with DENSE lanes, written to a workspace store at the
// particle's own slot; part 2 (advance_kernel<..., SPLIT = true>) reads it
// back and does the deposit and the in-super-cell shift.  Included by
// particles.cu inside namespace kwb, after advance.cuh.
//
// Why two kernels (profiles/r02_advance_ncu.md): the fused advance is
// issue/latency-bound at 16 warps/SM because the 54 register accumulators
// of the deposit window and the float64 push state share 128 registers,
// and because a warp walks its 32 cells' columns in lock step, so ~20 % of
// its lanes idle in the Poisson tails.  Here the float64 work runs without
// the window (fewer registers, more warps per SM) and each warp feeds its
// lanes from a compaction queue of its 32 cells' present slots, frame by
// frame, so all 32 lanes work until the warp's last batch.  The price is
// the workspace traffic: 28 B written here and read back in part 2.
//
// Reference arithmetic: identical to the fused kernel (gather6, push_move:
// pic/kernels.py:26-135 bit for bit).

#ifndef KWB_PUSH_MIN_BLOCKS
#define KWB_PUSH_MIN_BLOCKS 3
#endif

struct PushLayout {
    int tx, ty, tz, TV, boxx;
    size_t off_stage, off_queue, off_wrap, bytes;
};

template <typename F>
__host__ __device__ inline PushLayout push_layout(int scx, int scy, int scz) {
    PushLayout L;
    L.tx = scx + 2; L.ty = scy + 2; L.tz = scz + 2; L.TV = L.tx * L.ty * L.tz;
    constexpr int x0 = sizeof(F) == 4 ? 4 : 2, vec = 16 / (int)sizeof(F);
    L.boxx = (L.tx + x0 - 1 + vec - 1) / vec * vec;
    size_t o = (size_t)6 * L.TV * sizeof(double);
    o = (o + 127) & ~size_t(127);
    L.off_stage = o;
    o += (size_t)6 * L.boxx * L.ty * L.tz * sizeof(F);
    o = (o + 15) & ~size_t(15);
    L.off_queue = o;
    o += (size_t)kWarps * 64 * sizeof(int);
    L.off_wrap = o;
    o += (size_t)(L.tx + L.ty + L.tz) * sizeof(int);
    L.bytes = (o + 15) & ~size_t(15);
    return L;
}

template <typename F, int SX, int SY, int SZ>
__global__ void __launch_bounds__(kMaxCells, KWB_PUSH_MIN_BLOCKS)
push_kernel(Geo g, kwb_species sp, StoreT<F> in, StoreT<F> ws, FieldPtrs fp,
            const __grid_constant__ CUtensorMap tm_eb, int tma) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t s_mbar;
    const int scx = SX ? SX : g.scx, scy = SY ? SY : g.scy, scz = SZ ? SZ : g.scz;
    const int V = scx * scy * scz;
    const PushLayout L = push_layout<F>(scx, scy, scz);
    const int K = in.frames;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const bool owner = t < V;
    const int sc = blockIdx.x;
    const int bx = sc % g.gx, by = (sc / g.gx) % g.gy, bz = sc / (g.gx * g.gy);
    const int orgx = bx * scx, orgy = by * scy, orgz = bz * scz;

    const int64_t col = (int64_t)sc * V + t;
    const int f = owner ? in.front[col] : 0, b = owner ? in.back[col] : 0;
    if (__syncthreads_or(f + b) == 0) return;

    double *ebd = reinterpret_cast<double *>(smem_raw);
    int *wtx = reinterpret_cast<int *>(smem_raw + L.off_wrap);
    int *wty = wtx + L.tx, *wtz = wty + L.ty;
    int *wq = reinterpret_cast<int *>(smem_raw + L.off_queue) + wid * 64;

    // ---- E/B tile + 1 guard (TMA off the periodic seams, else indexed) -----
    const bool interior = bx >= 1 && bx + 2 <= g.gx && by >= 1 && by + 2 <= g.gy && bz >= 1 &&
                          bz + 2 <= g.gz;
    const bool use_tma = (tma & TMA_EB) && interior;
    constexpr int kX0 = sizeof(F) == 4 ? 4 : 2;
    F *stage = reinterpret_cast<F *>(smem_raw + L.off_stage);
    if (use_tma && t == 0) {
        mbar_init(&s_mbar, 1);
        fence_mbar_init();
        mbar_expect_tx(&s_mbar, (unsigned)(6 * L.boxx * L.ty * L.tz * sizeof(F)));
        tma_load_4d(stage, &tm_eb, orgx - kX0, orgy - 1, orgz - 1, 0, &s_mbar);
    }
    for (int i = t; i < L.tx; i += blockDim.x) wtx[i] = pymod(orgx - 1 + i, g.nx);
    for (int i = t; i < L.ty; i += blockDim.x) wty[i] = pymod(orgy - 1 + i, g.ny);
    for (int i = t; i < L.tz; i += blockDim.x) wtz[i] = pymod(orgz - 1 + i, g.nz);
    __syncthreads();
    const int total = 6 * L.TV, txy = L.tx * L.ty;
    if (use_tma) {
        mbar_wait(&s_mbar, 0);
        for (int i = t; i < total; i += blockDim.x) {
            const int c = i / L.TV, r = i - c * L.TV;
            const int d = r / txy, r2 = r - d * txy;
            const int y = r2 / L.tx, x = r2 - y * L.tx;
            ebd[i] = (double)stage[((c * L.tz + d) * L.ty + y) * L.boxx + x + kX0 - 1];
        }
    } else {
        for (int i = t; i < total; i += blockDim.x) {
            const int c = i / L.TV, r = i - c * L.TV;
            const int d = r / txy, r2 = r - d * txy;
            const int y = r2 / L.tx, x = r2 - y * L.tx;
            const void *sv = c == 0 ? fp.E[0] : c == 1 ? fp.E[1] : c == 2 ? fp.E[2]
                           : c == 3 ? fp.B[0] : c == 4 ? fp.B[1] : fp.B[2];
            ebd[i] = (double)__ldg((const F *)sv + ((int64_t)wtz[d] * g.ny + wty[y]) * g.nx + wtx[x]);
        }
    }
    __syncthreads();

    // ---- dense processing: each warp compacts its 32 cells' present slots,
    // frame by frame, into a queue and processes them 32 at a time ---------
    int fmax = f, bmax = b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        fmax = max(fmax, __shfl_xor_sync(0xffffffffu, fmax, o));
        bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    }
    const unsigned lt = (1u << lane) - 1u;
    int qn = 0, k = 0;
    for (;;) {
        while (qn < 32 && k < K) {   // warp-uniform
            if (k >= fmax && k < K - bmax) {   // the empty middle of every column
                k = K - bmax;
                continue;
            }
            const bool pres = owner && (k < f || k >= K - b);
            const unsigned m = __ballot_sync(0xffffffffu, pres);
            if (pres && KWB_IN(qn + __popc(m & lt) < 64)) wq[qn + __popc(m & lt)] = k * V + t;
            qn += __popc(m);
            ++k;
        }
        if (qn == 0) break;
        __syncwarp();
        const bool on = lane < qn;
        const int s_ = on ? wq[lane] : 0;
        const int rem = qn > 32 ? qn - 32 : 0;
        __syncwarp();
        if (lane < rem) wq[lane] = wq[32 + lane];
        __syncwarp();
        qn = rem;
        if (!on) continue;
        // the particle of slot (frame kk, cell c) of this super cell
        const int kk = s_ / V, c = s_ - kk * V;
        const int64_t q = ((int64_t)sc * K + kk) * V + c;
        const F ox = in.ox[q], oy = in.oy[q], oz = in.oz[q];
        const F ux = in.ux[q], uy = in.uy[q], uz = in.uz[q];
        const int lx = c % scx, ly = (c / scx) % scy, lz = c / (scx * scy);
        const double cxd = (double)(orgx + lx), cyd = (double)(orgy + ly), czd = (double)(orgz + lz);
        const double px = cxd + (double)ox, py = cyd + (double)oy, pz = czd + (double)oz;
        F e0, e1, e2, b0, b1, b2;
        gather6<F, double>(ebd, L.TV, L.tx, txy, (lz * L.ty + ly) * L.tx + lx, px, py, pz, cxd,
                           cyd, czd, e0, e1, e2, b0, b1, b2);
        F nux, nuy, nuz, nox, noy, noz;
        int dxi, dyi, dzi;
        push_move<F>(sp.qm_half_dt, sp.dt_d, e0, e1, e2, b0, b1, b2, ox, oy, oz, ux, uy, uz, nux,
                     nuy, nuz, nox, noy, noz, dxi, dyi, dzi);
        ws.ox[q] = nox; ws.oy[q] = noy; ws.oz[q] = noz;
        ws.ux[q] = nux; ws.uy[q] = nuy; ws.uz[q] = nuz;
        ws.w[q] = (F)pack_carries(dxi, dyi, dzi);   // small integer, exact in F
    }
}
