// Device construction plan: the degree draws of plan_jobs on the B200.
//
// Reference: proj/src/adjacency.cpp:29-71 (plan_jobs) and
// proj/include/synq/random.hpp:65-82 (geometric / binomial).
//
// The reference draws every (connection, source) degree from ONE master
// stream, derive_seed(seed, 0), connection by connection and source by
// source.  binomial(m, p) consumes hits + 1 draws: draw i contributes
// h_i = 1 + floor(log(u_i) / log1p(-p)) positions and the job ends at the
// first draw where the running sum reaches m + 1.  Only the segmentation is
// sequential; the draws' VALUES depend on their stream position alone.  So:
//
// * k_plan_draws: every thread jumps the xorshift128 state to its own chunk
//   of the stream (the generator is linear over GF(2): state_t = A^t state,
//   A^(L 2^k) precomputed) and writes h_i, clamped to m + 1 (a clamped draw
//   still ends its job at the same place), plus u64 sums per 256 draws.
//   CUDA's double log may differ from glibc's by an ulp, so a draw whose
//   quotient lies within a rigorous bound of an integer is listed and its h
//   recomputed on the host with glibc (k_plan_patch applies it).
// * k_plan_walk: one warp walks the job boundaries: 256-draw block sums find
//   the block a job ends in, one 256-draw load finds the draw; the next job
//   starts in the block already in registers.  About two dependent loads per
//   job instead of ~m p + 1 host logs.
// * The host loops over rounds of at most kPlanMaxDraws draws per connection
//   (an unfinished job is redone from its first draw in the next round) and
//   assembles the same construction_plan as plan_jobs.  Bit-identical to the
//   host plan by construction; tests/cpp/test_network.cu (case plan) checks it.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "synq/adjacency.hpp"
#include "synq/detail/cuda_util.hpp"
#include "synq/detail/device_graph.hpp"
#include "synq/random.hpp"

namespace synq {
namespace {

constexpr uint32_t kDrawsPerThread = 1024;  // L
constexpr uint32_t kJumpLevels = 15;        // A^(L 2^k), k < 15: up to 32768 threads per round
constexpr uint32_t kPlanMaxThreads = 1u << kJumpLevels;
constexpr uint64_t kPlanMaxDraws = static_cast<uint64_t>(kPlanMaxThreads) * kDrawsPerThread;
constexpr uint32_t kBlock = 256;  // draws per block sum
constexpr uint32_t kFlagCap = 1u << 16;

// 128x128 GF(2) matrix as 128 columns of 4 words (column b = A e_b)
struct gf2_matrix {
    uint32_t col[128][4];
};

__host__ __device__ inline void gf2_apply(const gf2_matrix& a, const uint32_t v[4], uint32_t out[4]) {
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    for (int b = 0; b < 128; ++b) {
        if ((v[b >> 5] >> (b & 31)) & 1u) {
            r0 ^= a.col[b][0];
            r1 ^= a.col[b][1];
            r2 ^= a.col[b][2];
            r3 ^= a.col[b][3];
        }
    }
    out[0] = r0, out[1] = r1, out[2] = r2, out[3] = r3;
}

gf2_matrix gf2_mul(const gf2_matrix& a, const gf2_matrix& b) {
    gf2_matrix c;
    for (int k = 0; k < 128; ++k) gf2_apply(a, b.col[k], c.col[k]);
    return c;
}

// one xorshift step as a matrix: column b = step(e_b)
gf2_matrix step_matrix() {
    gf2_matrix m;
    for (int b = 0; b < 128; ++b) {
        uint32_t s[4] = {0, 0, 0, 0};
        s[b >> 5] = 1u << (b & 31);
        xorshift r;
        r.load(s);
        r();
        r.save(m.col[b]);
    }
    return m;
}

// host jump table: pow2[k] = M^(2^k), k < 10 + kJumpLevels
struct jump_table {
    std::vector<gf2_matrix> pow2;
    jump_table() {
        pow2.push_back(step_matrix());
        for (int k = 1; k < 10 + static_cast<int>(kJumpLevels); ++k) pow2.push_back(gf2_mul(pow2.back(), pow2.back()));
    }
    void advance(uint32_t s[4], uint64_t n) const {
        for (size_t k = 0; n; ++k, n >>= 1) {
            if (!(n & 1)) continue;
            if (k >= pow2.size()) throw std::logic_error("plan jump out of range");
            uint32_t t[4];
            gf2_apply(pow2[k], s, t);
            std::memcpy(s, t, sizeof t);
        }
    }
};
static_assert(kDrawsPerThread == 1024, "jump table starts at M^(2^10)");

// h = 1 + floor(log(u) / denom), clamped to cap (= m + 1); flags quotients
// within 8 ulp of an integer (device log <= 1 ulp, glibc log <= 1 ulp, one
// rounding each side for the division)
__global__ void __launch_bounds__(256) k_plan_draws(const gf2_matrix* __restrict__ jump, uint4 base, uint32_t threads,
                                                    double denom, uint32_t cap, uint32_t* __restrict__ h,
                                                    unsigned long long* __restrict__ bsum,
                                                    uint2* __restrict__ flags, unsigned* __restrict__ nflags) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= threads) return;
    uint32_t s[4] = {base.x, base.y, base.z, base.w};
    for (uint32_t k = 0; k < kJumpLevels; ++k) {
        if ((t >> k) & 1u) {
            uint32_t o[4];
            gf2_apply(jump[k], s, o);
            s[0] = o[0], s[1] = o[1], s[2] = o[2], s[3] = o[3];
        }
    }
    xorshift r;
    r.load(s);
    const uint64_t first = static_cast<uint64_t>(t) * kDrawsPerThread;
    unsigned long long acc = 0;
    for (uint32_t i = 0; i < kDrawsPerThread; ++i) {
        const uint32_t x = r();
        const double u = (static_cast<double>(x) + 1.0) * 0x1p-32;
        const double q = log(u) / denom;
        const double f = floor(q);
        const double tol = fabs(q) * 0x1p-49 + 0x1p-1000;
        if (q - f < tol || (f + 1.0) - q < tol) {
            const unsigned slot = atomicAdd(nflags, 1u);
            if (slot < kFlagCap) flags[slot] = make_uint2(static_cast<uint32_t>(first + i), x);
        }
        const uint32_t hv = f >= static_cast<double>(cap) ? cap : static_cast<uint32_t>(f) + 1u;
        const uint32_t hc = hv > cap ? cap : hv;
        h[first + i] = hc;
        acc += hc;
        if ((i + 1) % kBlock == 0) {
            bsum[(first + i) / kBlock] = acc;
            acc = 0;
        }
    }
}

__global__ void k_plan_patch(const uint2* __restrict__ fix, uint32_t n, uint32_t* __restrict__ h,
                             unsigned long long* __restrict__ bsum) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t i = fix[j].x, v = fix[j].y;
    const uint32_t old = h[i];
    h[i] = v;
    atomicAdd(&bsum[i / kBlock], static_cast<unsigned long long>(v) - static_cast<unsigned long long>(old));
}

// lane l holds draws 8l .. 8l+7 of a 256-draw block
__device__ inline void load_block(const uint32_t* h, uint64_t blk, uint32_t lane, uint32_t v[8]) {
    const uint4* p = reinterpret_cast<const uint4*>(h + blk * kBlock) + lane * 2;
    const uint4 a = p[0], b = p[1];
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}

__device__ inline unsigned long long warp_incl_u64(unsigned long long x, uint32_t lane) {
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    return x;
}

// In the 256-draw block held in v (draws from index `from` on), find the
// draw where the running sum reaches `need`.  Returns the in-block index, or
// kBlock with `need` reduced by the block's (masked) total.
__device__ inline uint32_t find_in_block(const uint32_t v[8], uint32_t from, unsigned long long& need,
                                         uint32_t lane) {
    unsigned long long mine = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e)
        if (lane * 8 + e >= from) mine += v[e];
    const unsigned long long incl = warp_incl_u64(mine, lane);
    const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
    if (!hit) {
        need -= __shfl_sync(0xffffffffu, incl, 31);
        return kBlock;
    }
    const uint32_t fl = __ffs(hit) - 1;
    uint32_t pos = 0;
    if (lane == fl) {
        unsigned long long run = incl - mine;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (lane * 8 + e < from) continue;
            run += v[e];
            if (run >= need) {
                pos = lane * 8 + e;
                break;
            }
        }
    }
    return __shfl_sync(0xffffffffu, pos, fl);
}

// result[0] = jobs completed, result[1] = first draw of the next job
__global__ void k_plan_walk(const uint32_t* __restrict__ h, const unsigned long long* __restrict__ bsum,
                            uint64_t nblocks, uint32_t jobs, unsigned long long target,
                            uint32_t* __restrict__ hits, unsigned long long* __restrict__ result) {
    const uint32_t lane = threadIdx.x & 31;
    uint64_t start = 0;
    uint32_t done = 0;
    uint32_t v[8];
    uint64_t cached = ~0ull;
    // block-sum window prefetched with the block a job ends in: the next
    // job starts there, so its window (blocks pf_base ..) is already loaded
    unsigned long long pf = 0;
    uint64_t pf_base = ~0ull;
    while (done < jobs) {
        unsigned long long need = target;
        uint64_t blk = start / kBlock;
        if (blk >= nblocks) break;
        if (blk != cached) {
            load_block(h, blk, lane, v);
            cached = blk;
        }
        uint32_t at = find_in_block(v, static_cast<uint32_t>(start % kBlock), need, lane);
        bool ok = at < kBlock;
        while (!ok) {
            // skip whole blocks with the block sums, 32 at a time
            ++blk;
            if (blk >= nblocks) break;
            const unsigned long long bs =
                blk == pf_base ? pf : (blk + lane < nblocks ? bsum[blk + lane] : 0ull);
            const unsigned long long incl = warp_incl_u64(bs, lane);
            const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
            if (!hit) {
                need -= __shfl_sync(0xffffffffu, incl, 31);
                blk += 31;
                continue;
            }
            const uint32_t fl = __ffs(hit) - 1;
            need -= __shfl_sync(0xffffffffu, incl - bs, fl);
            blk += fl;
            load_block(h, blk, lane, v);
            pf_base = blk + 1;
            pf = pf_base + lane < nblocks ? bsum[pf_base + lane] : 0ull;
            cached = blk;
            at = find_in_block(v, 0, need, lane);
            ok = true;  // the block sum says it ends here
        }
        if (!ok) break;
        const uint64_t end = blk * kBlock + at;
        if (lane == 0) hits[done] = static_cast<uint32_t>(end - start);
        ++done;
        start = end + 1;
    }
    if (lane == 0) {
        result[0] = done;
        result[1] = start;
    }
}

}  // namespace

construction_plan plan_jobs_device(const network_desc& desc, uint64_t seed, uint32_t pitch_align,
                                   cudaStream_t stream) {
    const auto t_begin = std::chrono::steady_clock::now();
    static const jump_table jt;
    construction_plan plan;
    const uint32_t n = desc.neuron_count();
    plan.out_degree.assign(n, 0);

    std::vector<uint64_t> first(static_cast<size_t>(n) + 1, 0);
    for (const auto& c : desc.connections) {
        auto [sa, sb] = desc.id_range(c.src);
        for (uint32_t s = sa; s < sb; ++s) ++first[s + 1];
    }
    std::partial_sum(first.begin(), first.end(), first.begin());
    plan.jobs.resize(first[n]);
    std::vector<uint32_t> filled(n, 0);

    dev_array<gf2_matrix> djump(kJumpLevels);
    djump.upload(jt.pow2.data() + 10, kJumpLevels, stream);
    dev_array<uint32_t> h;
    dev_array<unsigned long long> bsum;
    dev_array<uint2> flags(kFlagCap);
    dev_array<unsigned> nflags(1);
    dev_array<unsigned long long> result(2);
    dev_array<uint2> fix(kFlagCap);
    dev_array<uint32_t> dhits;

    xorshift master(derive_seed(seed, 0));
    uint32_t state[4];
    master.save(state);
    std::vector<uint32_t> hits;
    std::vector<uint2> fl;
    const char* prof_env = std::getenv("SYNQ_PLAN_PROFILE");
    const bool prof = prof_env && std::atoi(prof_env) != 0;
    double t_draw = 0, t_walk = 0, t_pre = 0, t_conn = 0;
    {
        SYNQ_CUDA(cudaStreamSynchronize(stream));
        t_pre = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_begin).count();
    }
    const auto t_loop = std::chrono::steady_clock::now();
    uint64_t rounds = 0, guarded = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };

    for (const auto& c : desc.connections) {
        auto [sa, sb] = desc.id_range(c.src);
        auto [ta, tb] = desc.id_range(c.dst);
        const uint32_t ns = sb - sa, m = tb - ta;
        hits.assign(ns, 0);
        // binomial's no-draw cases (random.hpp:74-76)
        if (c.p >= 1.0 && m != 0) hits.assign(ns, m);
        if (!(c.p <= 0.0 || m == 0 || c.p >= 1.0) && ns) {
            if (m == 0xffffffffu) throw std::invalid_argument("plan: population too large");
            const double denom = std::log1p(-c.p);
            const uint32_t cap = m + 1;
            dhits.resize(ns);
            uint32_t done = 0;
            double grow = 1.05;
            while (done < ns) {
                const double expect = (ns - done) * (static_cast<double>(m) * c.p + 1.0) * grow + 4096.0;
                const uint32_t threads = static_cast<uint32_t>(
                    std::min<double>(kPlanMaxThreads, std::ceil(expect / kDrawsPerThread)));
                const uint64_t draws = static_cast<uint64_t>(threads) * kDrawsPerThread;
                if (h.size() < draws) {
                    h.resize(draws);
                    bsum.resize(draws / kBlock);
                }
                const auto tp0 = now();
                nflags.zero(stream);
                k_plan_draws<<<(threads + 255) / 256, 256, 0, stream>>>(
                    djump.get(), make_uint4(state[0], state[1], state[2], state[3]), threads, denom, cap, h.get(),
                    bsum.get(), flags.get(), nflags.get());
                SYNQ_CUDA(cudaGetLastError());
                unsigned nf = 0;
                nflags.download(&nf, 1, stream);
                SYNQ_CUDA(cudaStreamSynchronize(stream));
                const auto tp1 = now();
                t_draw += std::chrono::duration<double>(tp1 - tp0).count();
                ++rounds;
                guarded += nf;
                if (nf > kFlagCap) throw std::runtime_error("plan: too many rounding-guard draws");
                if (nf) {
                    // the reference's own arithmetic (geometric, random.hpp:69-72)
                    fl.resize(nf);
                    flags.download(fl.data(), nf, stream);
                    SYNQ_CUDA(cudaStreamSynchronize(stream));
                    for (auto& f : fl) {
                        const double u = (static_cast<double>(f.y) + 1.0) * 0x1p-32;
                        const uint64_t g = static_cast<uint64_t>(std::floor(std::log(u) / denom));
                        f.y = g >= cap ? cap : static_cast<uint32_t>(g) + 1u;
                    }
                    fix.upload(fl.data(), nf, stream);
                    k_plan_patch<<<(nf + 255) / 256, 256, 0, stream>>>(fix.get(), nf, h.get(), bsum.get());
                    SYNQ_CUDA(cudaGetLastError());
                }
                k_plan_walk<<<1, 32, 0, stream>>>(h.get(), bsum.get(), draws / kBlock, ns - done, cap,
                                                  dhits.get() + done, result.get());
                SYNQ_CUDA(cudaGetLastError());
                unsigned long long res[2];
                result.download(res, 2, stream);
                SYNQ_CUDA(cudaStreamSynchronize(stream));
                t_walk += std::chrono::duration<double>(now() - tp1).count();
                if (res[0] == 0) {
                    if (threads == kPlanMaxThreads) throw std::runtime_error("plan: job longer than a round");
                    grow *= 4.0;
                } else {
                    grow = 1.05;
                }
                done += static_cast<uint32_t>(res[0]);
                jt.advance(state, res[1]);
            }
            dhits.download(hits.data(), ns, stream);
            SYNQ_CUDA(cudaStreamSynchronize(stream));
        }
        for (uint32_t s = sa; s < sb; ++s) {
            const uint32_t k = hits[s - sa];
            plan.out_degree[s] += k;
            plan.jobs[first[s] + filled[s]++] = construction_job{k, ta, tb, 0};
        }
    }
    t_conn = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_loop).count();
    if (prof)
        std::fprintf(stderr,
                     "plan_jobs_device: setup %.3f s, connections %.3f s (%llu rounds, draws %.3f s, walk %.3f s), "
                     "%llu guarded draws\n",
                     t_pre, t_conn, static_cast<unsigned long long>(rounds), t_draw, t_walk,
                     static_cast<unsigned long long>(guarded));
    for (uint32_t d : plan.out_degree) plan.deg_max = std::max(plan.deg_max, d);
    if (pitch_align == 0) pitch_align = 1;
    plan.row_pitch = (plan.deg_max + pitch_align - 1) / pitch_align * pitch_align;
    for (uint32_t s = 0; s < n; ++s) {
        uint64_t o = static_cast<uint64_t>(s) * plan.row_pitch;
        for (uint64_t q = first[s]; q < first[s + 1]; ++q) {
            plan.jobs[q].o = o;
            o += plan.jobs[q].n;
            plan.total_edges += plan.jobs[q].n;
        }
    }
    return plan;
}

}  // namespace synq
