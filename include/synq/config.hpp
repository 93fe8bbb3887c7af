#pragma once
// Build-wide switches for the B200 synq engine.
//
// SYNQ_HD marks functions that run on both the host and the device.  Model
// callbacks (init / update / receive / init_synapse / update_synapse) are
// executed inside sm_100a kernels, so user-defined models annotate them with
// SYNQ_HD — the one source change the device engine asks of a model written
// against the reference API (proj/include/synq/engine.hpp:25-42).
#if defined(__CUDACC__)
#define SYNQ_HD __host__ __device__ __forceinline__
#define SYNQ_DEV __device__ __forceinline__
#else
#define SYNQ_HD inline
#define SYNQ_DEV inline
#endif

#if defined(__CUDA_ARCH__)
#define SYNQ_ON_DEVICE 1
#else
#define SYNQ_ON_DEVICE 0
#endif
