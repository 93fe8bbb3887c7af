// Network construction on the B200.
//
// Reference: proj/src/adjacency.cpp:29-109 (plan_jobs / expand_jobs /
// build_adjacency) and proj/include/synq/adjacency.hpp:112-163
// (sorted_random).
//
// * plan_jobs: ONE sequential binomial stream (derive_seed(seed, 0)) whose
//   draw positions are data dependent.  The host restatement below is kept as
//   the SYNQ_HOST_PLAN=1 path and the check; the default is the device plan
//   (csrc/plan.cu): the same stream jumped ahead per thread, glibc-guarded.
// * expansion runs on the device, one thread per job.  Each thread replays
//   its job's xorshift stream twice (pass 1: the exclusive-sum total, pass 2:
//   the outputs) with the same left-to-right double summation as the
//   reference, and writes directly into the job's final position inside the
//   row.  A source's jobs target disjoint populations, so ordering the jobs of
//   a row by range start yields the sorted row the reference gets from
//   std::sort — no sort pass on the device.
// * exactness guard: CUDA's double log and glibc's may differ by an ulp.  A
//   rigorous bound on the resulting error of v = prefix/total*scale is
//   computed per job; any output whose v+0.5 lies within that bound of an
//   integer flags the job, and flagged jobs are recomputed on the host with
//   glibc and patched in.  The table is therefore bit-identical to the
//   reference's.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <fstream>
#include <numeric>
#include <stdexcept>
#include <mutex>
#include <thread>
#include <vector>

#include "synq/adjacency.hpp"
#include "synq/detail/device_graph.hpp"
#include "synq/random.hpp"

namespace synq {

// ------------------------------------------------------------ host mirror
adjacency_list::adjacency_list(uint32_t neurons, uint32_t deg_max, uint32_t row_pitch)
    : neurons_(neurons), deg_max_(deg_max), pitch_(row_pitch) {
    cells_.assign(static_cast<size_t>(neurons) * row_pitch, sentinel);
    degree_.assign(neurons, 0);
}

adjacency_list::adjacency_list(uint32_t neurons, uint32_t deg_max, uint32_t row_pitch,
                               std::vector<uint32_t> cells, std::vector<uint32_t> degree)
    : neurons_(neurons), deg_max_(deg_max), pitch_(row_pitch), cells_(std::move(cells)),
      degree_(std::move(degree)) {
    edges_ = 0;
    for (uint32_t d : degree_) edges_ += d;
}

std::span<const uint32_t> adjacency_list::row(uint32_t id) const {
    if (id >= neurons_) throw std::out_of_range("adjacency row id out of range");
    return {cells_.data() + static_cast<size_t>(id) * pitch_, degree_[id]};
}

std::span<const uint32_t> adjacency_list::raw_row(uint32_t id) const {
    if (id >= neurons_) throw std::out_of_range("adjacency row id out of range");
    return {cells_.data() + static_cast<size_t>(id) * pitch_, pitch_};
}

// binary format of adjacency.cpp:122-163: u32 neurons, pitch, deg_max,
// sentinel, then neurons*pitch u32 cells; degrees are recovered on load
void adjacency_list::dump(std::ostream& out) const {
    const uint32_t hdr[4] = {neurons_, pitch_, deg_max_, sentinel};
    out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
    out.write(reinterpret_cast<const char*>(cells_.data()),
              static_cast<std::streamsize>(cells_.size() * sizeof(uint32_t)));
}

adjacency_list adjacency_list::load(std::istream& in) {
    uint32_t hdr[4] = {0, 0, 0, 0};
    in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
    if (!in || hdr[3] != sentinel) throw std::runtime_error("adjacency load: bad header");
    adjacency_list adj(hdr[0], hdr[2], hdr[1]);
    in.read(reinterpret_cast<char*>(adj.cells_.data()),
            static_cast<std::streamsize>(adj.cells_.size() * sizeof(uint32_t)));
    if (!in) throw std::runtime_error("adjacency load: truncated data");
    adj.edges_ = 0;
    for (uint32_t r = 0; r < adj.neurons_; ++r) {
        const uint32_t* row = adj.cells_.data() + static_cast<size_t>(r) * adj.pitch_;
        uint32_t d = 0;
        while (d < adj.pitch_ && row[d] != sentinel) ++d;
        adj.degree_[r] = d;
        adj.edges_ += d;
    }
    return adj;
}

void adjacency_list::save_file(const std::string& path) const {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    dump(out);
}

adjacency_list adjacency_list::load_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open: " + path);
    return load(in);
}

// ------------------------------------------------------------------ plan
construction_plan plan_jobs(const network_desc& desc, uint64_t seed, uint32_t pitch_align) {
    construction_plan plan;
    const uint32_t n = desc.neuron_count();
    plan.out_degree.assign(n, 0);
    xorshift master(derive_seed(seed, 0));

    // jobs are emitted source-major in connection order; count them first
    std::vector<uint64_t> first(static_cast<size_t>(n) + 1, 0);
    for (const auto& c : desc.connections) {
        auto [sa, sb] = desc.id_range(c.src);
        for (uint32_t s = sa; s < sb; ++s) ++first[s + 1];
    }
    std::partial_sum(first.begin(), first.end(), first.begin());
    plan.jobs.resize(first[n]);
    std::vector<uint32_t> filled(n, 0);

    // the degree draws themselves consume the master stream connection by
    // connection, source by source (adjacency.cpp:41-51)
    for (const auto& c : desc.connections) {
        auto [sa, sb] = desc.id_range(c.src);
        auto [ta, tb] = desc.id_range(c.dst);
        for (uint32_t s = sa; s < sb; ++s) {
            const uint32_t k = binomial(tb - ta, c.p, master);
            plan.out_degree[s] += k;
            plan.jobs[first[s] + filled[s]++] = construction_job{k, ta, tb, 0};
        }
    }
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

// ------------------------------------------------------------- expansion
namespace {

struct dev_job {
    uint32_t n, a, b;
    uint32_t nl;     // outputs inside the target range [tlo, thi) (= n for a full build)
    uint64_t o;      // final (sorted) offset of the job's first output
    uint64_t index;  // position in plan order: the stream is derive_seed(seed, index + 1)
};

// rigorous per-job bound on |v_device - v_host| for v = prefix/total*scale
// when the two logs may differ by <= 2 ulp (see file comment)
__host__ __device__ inline double tie_guard(uint32_t n, double scale) {
    return 2.0 * scale * (6.0 * (n + 2.0) + 24.0) * 0x1p-52 + 1e-12;
}

// mode 0: write the job's outputs inside [tlo, thi) (at most job.nl of them)
// to cells + job.o; mode 1: count them into lcount[j] (shard sub-rows).  Jobs
// whose range lies inside [tlo, thi) need no replay to be counted.
__global__ void k_expand(const dev_job* __restrict__ jobs, uint64_t njobs, uint64_t seed, uint32_t tlo,
                         uint32_t thi, int mode, uint32_t* __restrict__ cells, uint32_t* __restrict__ lcount,
                         uint64_t* __restrict__ flagged, unsigned long long* __restrict__ nflagged,
                         uint64_t flag_cap) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < njobs;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const dev_job job = jobs[j];
        const bool inside = job.a >= tlo && job.b <= thi;
        if (mode == 1) {
            if (inside || job.n == 0 || job.b <= tlo || job.a >= thi) {
                lcount[j] = inside ? job.n : 0u;
                continue;
            }
        } else if (job.nl == 0) {
            continue;
        }
        const uint64_t stream = derive_seed(seed, job.index + 1);
        // pass 1: total = sum of the first n+1 exponentials, left to right
        xorshift r(stream);
        double total = 0.0;
        for (uint32_t i = 0; i <= job.n; ++i) total += -log(r.uniform01());
        if (total <= 0.0) total = 1.0;
        const double scale = static_cast<double>(job.b - job.a - job.n);
        const double guard = tie_guard(job.n, scale);
        // pass 2: replay the stream, emit a + round_half_up(prefix/total*scale) + i
        r = xorshift(stream);
        double prefix = 0.0;
        bool close = false;
        uint32_t* out = cells + job.o;
        uint32_t k = 0;
        for (uint32_t i = 0; i < job.n; ++i) {
            prefix += -log(r.uniform01());
            const double v = prefix / total * scale;
            const double f = floor(v + 0.5);
            const double d = (v + 0.5) - f;
            close |= (d < guard) || (1.0 - d < guard);
            const uint32_t t = job.a + static_cast<uint32_t>(f) + i;
            if (t >= tlo && t < thi) {
                if (mode == 0 && k < job.nl) out[k] = t;
                ++k;
            }
        }
        if (mode == 1) lcount[j] = k;
        if (close) {
            const unsigned long long slot = atomicAdd(nflagged, 1ull);
            if (slot < flag_cap) flagged[slot] = j;
        }
    }
}

__global__ void k_in_degree(const uint32_t* __restrict__ cells, const uint32_t* __restrict__ degree,
                            uint32_t neurons, uint32_t pitch, uint32_t* __restrict__ indeg) {
    // one warp per row: rows are short relative to the grid, lanes stride the row
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t s = warp; s < neurons; s += nwarps) {
        const uint32_t d = degree[s];
        const uint32_t* row = cells + s * pitch;
        for (uint32_t k = lane; k < d; k += 32) atomicAdd(&indeg[row[k]], 1u);
    }
}

__global__ void k_splits(const uint32_t* __restrict__ cells, const uint32_t* __restrict__ degree,
                         uint32_t neurons, uint32_t pitch, const uint32_t* __restrict__ tile_lo,
                         uint32_t tiles, uint32_t* __restrict__ split) {
    const uint64_t total = static_cast<uint64_t>(neurons) * (tiles + 1);
    for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
         x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t s = x / (tiles + 1);
        const uint32_t c = static_cast<uint32_t>(x % (tiles + 1));
        const uint32_t d = degree[s];
        // lower_bound of the boundary; the last boundary of a shard is not
        // the end of the row (its targets stop at the shard's range)
        const uint32_t key = tile_lo[c];
        const uint32_t* row = cells + s * pitch;
        uint32_t lo = 0, hi = d;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (row[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        const uint32_t pos = lo;
        split[x] = pos;
    }
}

int grid_for(uint64_t work, int block) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (work + block - 1) / block;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(want, 32ull * sms)));
}

}  // namespace

namespace {

// Recompute the listed jobs on the host with glibc (the reference's exact
// path) on all host cores, in chunks of at most kChunkWords staged output
// words.  emit(i, outputs) receives job fl[i]'s in-range outputs (a
// contiguous run of the sorted job output) and the chunk's staging base; it
// runs on the calling thread after the chunk is complete, in list order.  A
// worker's exception (bad_alloc ...) is rethrown after the join, so guarded()
// maps it to a status instead of std::terminate.
template <class Emit>
void host_recompute(const std::vector<dev_job>& jobs, const std::vector<uint64_t>& fl, uint64_t seed,
                    uint32_t tlo, uint32_t thi, cudaStream_t stream, Emit&& emit) {
    constexpr uint64_t kChunkWords = uint64_t(1) << 24;  // 64 MB
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16));
    std::vector<uint32_t> stage;
    std::vector<uint64_t> at, len;  // staging offset / in-range outputs of each job of the chunk
    for (size_t q0 = 0; q0 < fl.size();) {
        size_t q1 = q0;
        uint64_t words = 0;
        at.clear();
        while (q1 < fl.size() && (q1 == q0 || words + jobs[fl[q1]].n <= kChunkWords)) {
            at.push_back(words);
            words += jobs[fl[q1]].n;
            ++q1;
        }
        stage.resize(std::max<uint64_t>(1, words));
        len.assign(q1 - q0, 0);
        std::atomic<size_t> next{q0};
        std::exception_ptr err;
        std::mutex err_mu;
        auto work = [&] {
            try {
                for (size_t i; (i = next.fetch_add(1)) < q1;) {
                    const dev_job& job = jobs[fl[i]];
                    xorshift r(derive_seed(seed, job.index + 1));
                    uint32_t* out = stage.data() + at[i - q0];
                    sorted_random(job.n, job.a, job.b, r, out);
                    // keep the outputs inside [tlo, thi), moved to the front
                    const uint32_t* lo = std::lower_bound(out, out + job.n, tlo);
                    const uint32_t* hi = std::lower_bound(lo, static_cast<const uint32_t*>(out + job.n), thi);
                    std::memmove(out, lo, static_cast<size_t>(hi - lo) * sizeof(uint32_t));
                    len[i - q0] = static_cast<uint64_t>(hi - lo);
                }
            } catch (...) {
                std::lock_guard<std::mutex> lk(err_mu);
                if (!err) err = std::current_exception();
                next.store(q1);
            }
        };
        std::vector<std::thread> pool;
        for (unsigned k = 1; k < nt && k < q1 - q0; ++k) pool.emplace_back(work);
        work();
        for (auto& th : pool) th.join();
        if (err) std::rethrow_exception(err);
        for (size_t i = q0; i < q1; ++i) emit(i, stage.data() + at[i - q0], len[i - q0]);
        SYNQ_CUDA(cudaStreamSynchronize(stream));  // the staging buffer is reused by the next chunk
        q0 = q1;
    }
}

// run k_expand over `jobs` and return the guard-flagged job indices (every
// job when more were flagged than listed: never expected)
std::vector<uint64_t> run_expand(const dev_array<dev_job>& djobs, size_t njobs, uint64_t seed, uint32_t tlo,
                                 uint32_t thi, int mode, uint32_t* cells, uint32_t* lcount, cudaStream_t stream) {
    const uint64_t flag_cap = 1u << 20;
    dev_array<uint64_t> flagged(flag_cap);
    dev_array<unsigned long long> nflag(1);
    nflag.zero(stream);
    if (njobs) {
        k_expand<<<grid_for(njobs, 128), 128, 0, stream>>>(djobs.get(), njobs, seed, tlo, thi, mode, cells, lcount,
                                                            flagged.get(), nflag.get(), flag_cap);
        SYNQ_CUDA(cudaGetLastError());
    }
    unsigned long long nf = 0;
    nflag.download(&nf, 1, stream);
    SYNQ_CUDA(cudaStreamSynchronize(stream));
    std::vector<uint64_t> fl(std::min<unsigned long long>(nf, flag_cap));
    flagged.download(fl.data(), fl.size(), stream);
    SYNQ_CUDA(cudaStreamSynchronize(stream));
    if (nf > flag_cap) {
        fl.resize(njobs);
        std::iota(fl.begin(), fl.end(), 0);
    } else {
        std::sort(fl.begin(), fl.end());
    }
    return fl;
}

}  // namespace

device_graph expand_device_graph(const construction_plan& plan, uint32_t neurons, uint64_t seed,
                                 cudaStream_t stream, uint32_t tlo, uint32_t thi, uint32_t pitch_align) {
    thi = std::min(thi, neurons);
    tlo = std::min(tlo, thi);
    const bool full = tlo == 0 && thi == neurons;
    device_graph g;
    g.neurons = neurons;
    g.target_lo = tlo;
    g.target_hi = thi;
    g.jobs = plan.jobs.size();

    // a row's non-empty jobs ordered by target-range start (a source's jobs
    // target disjoint populations, so this is the row's sorted order).  A
    // non-empty job's plan offset lies strictly inside its row, so
    // o / row_pitch is its source; empty jobs write nothing and are dropped,
    // and so are the jobs of a sub-row build whose range misses [tlo, thi).
    std::vector<dev_job> jobs;
    std::vector<uint32_t> row_of;
    jobs.reserve(plan.jobs.size());
    for (size_t q = 0; q < plan.jobs.size(); ++q) {
        const auto& pj = plan.jobs[q];
        if (pj.n == 0 || pj.b <= tlo || pj.a >= thi) continue;
        jobs.push_back(dev_job{pj.n, pj.a, pj.b, pj.n, 0, static_cast<uint64_t>(q)});
        row_of.push_back(static_cast<uint32_t>(pj.o / plan.row_pitch));
    }
    std::vector<size_t> order(jobs.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
        return row_of[x] != row_of[y] ? row_of[x] < row_of[y] : jobs[x].a < jobs[y].a;
    });
    {
        std::vector<dev_job> sj(jobs.size());
        std::vector<uint32_t> sr(jobs.size());
        for (size_t k = 0; k < order.size(); ++k) {
            sj[k] = jobs[order[k]];
            sr[k] = row_of[order[k]];
        }
        jobs.swap(sj);
        row_of.swap(sr);
    }
    dev_array<dev_job> djobs(std::max<size_t>(1, jobs.size()));
    const char* prof_env = std::getenv("SYNQ_PLAN_PROFILE");
    const bool prof = prof_env && std::atoi(prof_env) != 0;

    g.host_degree.assign(neurons, 0);
    if (full) {
        g.host_degree = plan.out_degree;
        g.host_degree.resize(neurons, 0);
        g.deg_max = plan.deg_max;
        g.pitch = plan.row_pitch;
        g.edges = plan.total_edges;
    } else {
        // sub-rows of a shard: count each job's outputs inside
        // [tlo, thi) on the device (exact for jobs inside the range; guard-
        // flagged straddling jobs are recounted on the host with glibc)
        djobs.upload(jobs.data(), jobs.size(), stream);
        dev_array<uint32_t> lcount(std::max<size_t>(1, jobs.size()));
        const std::vector<uint64_t> fl =
            run_expand(djobs, jobs.size(), seed, tlo, thi, 1, nullptr, lcount.get(), stream);
        std::vector<uint32_t> nl(jobs.size());
        lcount.download(nl.data(), nl.size(), stream);
        SYNQ_CUDA(cudaStreamSynchronize(stream));
        host_recompute(jobs, fl, seed, tlo, thi, stream,
                       [&](size_t i, const uint32_t*, uint64_t n) { nl[fl[i]] = static_cast<uint32_t>(n); });
        if (prof) std::fprintf(stderr, "expand [%u, %u): %zu jobs recounted on the host\n", tlo, thi, fl.size());
        size_t w = 0;
        for (size_t k = 0; k < jobs.size(); ++k) {
            if (nl[k] == 0) continue;
            jobs[w] = jobs[k];
            jobs[w].nl = nl[k];
            row_of[w] = row_of[k];
            g.host_degree[row_of[k]] += nl[k];
            g.edges += nl[k];
            ++w;
        }
        jobs.resize(w);
        row_of.resize(w);
        for (uint32_t d : g.host_degree) g.deg_max = std::max(g.deg_max, d);
        const uint32_t align = std::max<uint32_t>(1, pitch_align);
        g.pitch = (g.deg_max + align - 1) / align * align;
    }
    // final offsets: the jobs of a row back to back
    for (size_t q = 0; q < jobs.size();) {
        size_t e = q + 1;
        while (e < jobs.size() && row_of[e] == row_of[q]) ++e;
        uint64_t o = static_cast<uint64_t>(row_of[q]) * g.pitch;
        for (size_t k = q; k < e; ++k) {
            jobs[k].o = o;
            o += jobs[k].nl;
        }
        q = e;
    }

    const size_t ncells = static_cast<size_t>(neurons) * g.pitch;
    g.cells.resize(std::max<size_t>(1, ncells));
    g.cells.fill_bytes(0xff, stream);  // sentinel padding
    g.degree.resize(std::max<uint32_t>(1, neurons));
    g.degree.upload(g.host_degree.data(), neurons, stream);
    djobs.upload(jobs.data(), jobs.size(), stream);
    const std::vector<uint64_t> fl =
        run_expand(djobs, jobs.size(), seed, tlo, thi, 0, g.cells.get(), nullptr, stream);
    if (prof) std::fprintf(stderr, "expand: %zu jobs recomputed on the host\n", fl.size());
    // host fix-up of guard-flagged jobs: glibc log, the reference's exact path
    host_recompute(jobs, fl, seed, tlo, thi, stream, [&](size_t i, const uint32_t* out, uint64_t n) {
        const dev_job& job = jobs[fl[i]];
        if (n != job.nl) throw std::logic_error("expand: host recount differs from the job's sub-row count");
        SYNQ_CUDA(cudaMemcpyAsync(g.cells.get() + job.o, out, n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    });
    g.tie_fixups = fl.size();
    return g;
}

device_graph build_device_graph(const network_desc& desc, uint64_t seed, uint32_t pitch_align,
                                cudaStream_t stream, uint32_t tlo, uint32_t thi) {
    // both plans are identical; pick the cheaper: the host spends ~5.5 ns per
    // master-stream draw (m p + 1 per job), the device walk ~1 us per job
    // (B200: Brunel 1e9 11.6 s host vs 0.32 s device; 604k tiny jobs 0.07 s
    // host vs 0.5 s device)
    double draws = 0, jobs = 0;
    for (const auto& c : desc.connections) {
        auto [sa, sb] = desc.id_range(c.src);
        auto [ta, tb] = desc.id_range(c.dst);
        jobs += sb - sa;
        if (c.p > 0.0 && c.p < 1.0) draws += (sb - sa) * ((tb - ta) * c.p + 1.0);
    }
    const char* host = std::getenv("SYNQ_HOST_PLAN");
    const bool on_host = host ? std::atoi(host) != 0 : draws * 5.5e-9 < jobs * 1.0e-6 + 2e-3;
    return expand_device_graph(on_host ? plan_jobs(desc, seed, pitch_align)
                                       : plan_jobs_device(desc, seed, pitch_align, stream),
                               desc.neuron_count(), seed, stream, tlo, thi, pitch_align);
}

adjacency_list download_graph(const device_graph& g, cudaStream_t stream) {
    std::vector<uint32_t> cells(static_cast<size_t>(g.neurons) * g.pitch);
    g.cells.download(cells.data(), cells.size(), stream);
    SYNQ_CUDA(cudaStreamSynchronize(stream));
    return adjacency_list(g.neurons, g.deg_max, g.pitch, std::move(cells), g.host_degree);
}

device_graph upload_graph(const adjacency_list& adj, cudaStream_t stream) {
    device_graph g;
    g.neurons = adj.neuron_count();
    g.target_hi = g.neurons;
    g.deg_max = adj.deg_max();
    g.pitch = adj.row_pitch();
    g.edges = adj.edge_count();
    g.host_degree.assign(adj.degrees(), adj.degrees() + g.neurons);
    g.cells.resize(static_cast<size_t>(g.neurons) * g.pitch);
    g.cells.upload(adj.cells(), g.cells.size(), stream);
    g.degree.resize(g.neurons);
    g.degree.upload(g.host_degree.data(), g.neurons, stream);
    SYNQ_CUDA(cudaStreamSynchronize(stream));
    return g;
}

std::vector<uint32_t> in_degrees(const device_graph& g, cudaStream_t stream) {
    std::vector<uint32_t> out(g.neurons, 0);
    if (!g.neurons) return out;
    dev_array<uint32_t> indeg(g.neurons);
    indeg.zero(stream);
    if (g.edges) {
        k_in_degree<<<grid_for(static_cast<uint64_t>(g.neurons) * 32, 256), 256, 0, stream>>>(
            g.cells.get(), g.degree.get(), g.neurons, g.pitch, indeg.get());
        SYNQ_CUDA(cudaGetLastError());
    }
    indeg.download(out.data(), g.neurons, stream);
    SYNQ_CUDA(cudaStreamSynchronize(stream));
    return out;
}

void build_splits(const device_graph& g, const std::vector<uint32_t>& tile_lo,
                  dev_array<uint32_t>& split, cudaStream_t stream) {
    const uint32_t tiles = static_cast<uint32_t>(tile_lo.size()) - 1;
    dev_array<uint32_t> dlo(tile_lo.size());
    dlo.upload(tile_lo.data(), tile_lo.size(), stream);
    split.resize(std::max<size_t>(1, static_cast<size_t>(g.neurons) * (tiles + 1)));
    const uint64_t work = static_cast<uint64_t>(g.neurons) * (tiles + 1);
    if (work) {
        k_splits<<<grid_for(work, 256), 256, 0, stream>>>(g.cells.get(), g.degree.get(), g.neurons,
                                                           g.pitch, dlo.get(), tiles, split.get());
        SYNQ_CUDA(cudaGetLastError());
    }
    SYNQ_CUDA(cudaStreamSynchronize(stream));
}

// Receive-window bitmaps (pipeline.cuh, bitmap delivery): row s holds, for
// every local CTA c, wq uint4 (= 128 * wq bits) whose bit k is set iff
// target window_lo[c] + k is in row s.  One CTA assembles a row in shared
// memory (targets arrive sorted, so neighbouring threads hit neighbouring
// words) and writes it out with 16-byte stores.
__global__ void k_window_bitmaps(const uint32_t* __restrict__ cells, const uint32_t* __restrict__ degree,
                                 uint32_t neurons, uint32_t pitch, const uint32_t* __restrict__ tpos,
                                 uint32_t row_words, uint4* __restrict__ bm) {
    extern __shared__ __align__(16) uint32_t row[];
    for (uint32_t s = blockIdx.x; s < neurons; s += gridDim.x) {
        for (uint32_t w = threadIdx.x; w < row_words; w += blockDim.x) row[w] = 0;
        __syncthreads();
        const uint32_t d = degree[s];
        const uint32_t* r = cells + static_cast<uint64_t>(s) * pitch;
        for (uint32_t k = threadIdx.x; k < d; k += blockDim.x) {
            const uint32_t e = __ldg(tpos + __ldg(r + k));
            if (e != 0xffffffffu) atomicOr(&row[e >> 5], 1u << (e & 31));
        }
        __syncthreads();
        uint4* out = bm + static_cast<uint64_t>(s) * (row_words / 4);
        const uint4* rw = reinterpret_cast<const uint4*>(row);
        for (uint32_t q = threadIdx.x; q < row_words / 4; q += blockDim.x) out[q] = rw[q];
        __syncthreads();
    }
}

void build_window_bitmaps(const device_graph& g, const std::vector<uint32_t>& window_lo,
                          const std::vector<uint32_t>& window_hi, uint32_t wq, dev_array<uint4>& bm,
                          cudaStream_t stream) {
    const uint32_t C = static_cast<uint32_t>(window_lo.size());
    const uint32_t row_words = C * wq * 4;
    std::vector<uint32_t> tpos(std::max<uint32_t>(1, g.neurons), 0xffffffffu);
    for (uint32_t c = 0; c < C; ++c)
        for (uint32_t t = window_lo[c]; t < window_hi[c]; ++t) {
            const uint32_t k = t - window_lo[c];
            if (k >= wq * 128) throw std::invalid_argument("window bitmap: window wider than its row slice");
            tpos[t] = (c * wq * 4 + k / 32) << 5 | (k % 32);
        }
    dev_array<uint32_t> dpos(tpos.size());
    dpos.upload(tpos.data(), tpos.size(), stream);
    bm.resize(std::max<size_t>(1, static_cast<size_t>(g.neurons) * (row_words / 4)));
    if (g.neurons && row_words) {
        const size_t smem = size_t(row_words) * 4;
        if (smem > 48 * 1024)
            SYNQ_CUDA(cudaFuncSetAttribute(k_window_bitmaps, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
        int sms = 0, dev = 0;
        SYNQ_CUDA(cudaGetDevice(&dev));
        SYNQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const uint32_t grid = std::min<uint32_t>(g.neurons, static_cast<uint32_t>(sms) * 8);
        k_window_bitmaps<<<grid, 256, smem, stream>>>(g.cells.get(), g.degree.get(), g.neurons, g.pitch,
                                                      dpos.get(), row_words, bm.get());
        SYNQ_CUDA(cudaGetLastError());
    }
    SYNQ_CUDA(cudaStreamSynchronize(stream));
}

adjacency_list expand_jobs(const construction_plan& plan, uint32_t neurons, uint64_t seed,
                           thread_pool*) {
    device_graph g = expand_device_graph(plan, neurons, seed, nullptr, 0, neurons, 32);
    return download_graph(g, nullptr);
}

adjacency_list build_adjacency(const network_desc& desc, uint64_t seed, uint32_t pitch_align,
                               thread_pool*) {
    device_graph g = build_device_graph(desc, seed, pitch_align, nullptr);
    return download_graph(g, nullptr);
}

}  // namespace synq
