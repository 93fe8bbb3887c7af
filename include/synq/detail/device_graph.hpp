#pragma once
// Device-resident padded-ELL adjacency and the construction entry points
// implemented in libsynq (paper_1912_07423_b200/csrc/construct.cu).
//
// HBM layout: cells[neurons * pitch] u32, row-major, each row sorted and
// padded with 0xFFFFFFFF (pitch = deg_max rounded up to pitch_align, 32 by
// default = 128-byte rows); degree[neurons] u32.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "synq/adjacency.hpp"
#include "synq/detail/cuda_util.hpp"
#include "synq/network_desc.hpp"

namespace synq {

struct device_graph {
    uint32_t neurons = 0;
    uint32_t deg_max = 0;
    uint32_t pitch = 0;
    uint64_t edges = 0;
    uint64_t jobs = 0;
    uint64_t tie_fixups = 0;  // jobs recomputed on the host by the rounding guard
    // targets held: [target_lo, target_hi) (a shard's sub-rows, SURVEY.md 8e;
    // the whole id space otherwise).  deg_max / pitch / edges / degree are
    // those of the sub-rows.
    uint32_t target_lo = 0, target_hi = 0;
    dev_array<uint32_t> cells;
    dev_array<uint32_t> degree;
    std::vector<uint32_t> host_degree;

    uint64_t bytes() const { return cells.bytes() + degree.bytes(); }
};

// the degree plan of plan_jobs drawn on the device (csrc/plan.cu); the same
// construction_plan as the host plan_jobs, bit for bit
construction_plan plan_jobs_device(const network_desc& desc, uint64_t seed, uint32_t pitch_align,
                                   cudaStream_t stream);
// plan on the device (SYNQ_HOST_PLAN=1: on the host), expand on the device.
// [tlo, thi): keep only the targets in this range (every row's sub-row, still
// sorted; pitch = that sub-row maximum rounded up to pitch_align): the
// storage of one shard of a target-partitioned multi-GPU run.
device_graph build_device_graph(const network_desc& desc, uint64_t seed, uint32_t pitch_align,
                                cudaStream_t stream, uint32_t tlo = 0, uint32_t thi = 0xffffffffu);
device_graph expand_device_graph(const construction_plan& plan, uint32_t neurons, uint64_t seed,
                                 cudaStream_t stream, uint32_t tlo, uint32_t thi, uint32_t pitch_align);
// host mirror of a device graph
adjacency_list download_graph(const device_graph& g, cudaStream_t stream);
// upload a host table (adjacency_list::load) to the device
device_graph upload_graph(const adjacency_list& adj, cudaStream_t stream);
// in-degree histogram (device), for target partitioning
std::vector<uint32_t> in_degrees(const device_graph& g, cudaStream_t stream);
// split[s * (tiles + 1) + c] = first row position of row s whose target is
// >= tile_lo[c]  (tile_lo has tiles + 1 entries, the last = neurons)
void build_splits(const device_graph& g, const std::vector<uint32_t>& tile_lo,
                  dev_array<uint32_t>& split, cudaStream_t stream);

// receive-window bitmaps for the bitmap delivery of the pipelined engine:
// bm[s * C * wq + c * wq + q] (uint4) holds bits 128q .. 128q+127 of window c
// ([window_lo[c], window_hi[c]) target ids, at most 128 * wq wide) of row s
void build_window_bitmaps(const device_graph& g, const std::vector<uint32_t>& window_lo,
                          const std::vector<uint32_t>& window_hi, uint32_t wq, dev_array<uint4>& bm,
                          cudaStream_t stream);

}  // namespace synq
