/*
 * fourierbf_b200.h -- the C-ABI boundary of the B200 shiftable bilateral filter.
 *
 * Plain C: pointers, sizes and status codes, no C++ or torch types.  These
 * entry points replace the reference's hot path
 *   fourierbf::bilateral_fast   /root/reference/proj/include/fourierbf/bilateral.hpp:109-160
 *   fourierbf::convolve         /root/reference/proj/include/fourierbf/spatial.hpp:98-112
 * The reference's own C++ API (the headers under include/fourierbf/) is
 * implemented on top of them; INTEGRATION.md shows the ctypes binding.
 *
 * Errors follow the reference's conventions (bilateral.hpp:112-118,147-158):
 *   FBF_EINVAL   <-> std::invalid_argument (empty image; eps >= w0; bad sizes)
 *   FBF_EANOMALY <-> std::runtime_error "denominator collapsed at pixel (x, y)",
 *                    *bad_index = first offending row-major index
 * fbf_last_error() returns the thread's message for the last failing call.
 * All entry points are reentrant: no global mutable state besides a cached
 * per-device attribute table and the thread-local error string.
 */
#ifndef FOURIERBF_B200_H
#define FOURIERBF_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBF_OK 0
#define FBF_EINVAL 1
#define FBF_EANOMALY 2
#define FBF_ECUDA 3
#define FBF_EUNSUPPORTED 4

#define FBF_SPATIAL_GAUSSIAN 0 /* spatial.hpp:13 SpatialKind::gaussian */
#define FBF_SPATIAL_BOX 1      /* spatial.hpp:13 SpatialKind::box      */

#define FBF_RANGE_GAUSSIAN 0    /* kernels.hpp:12 RangeFamily::gaussian    */
#define FBF_RANGE_EXPONENTIAL 1 /* kernels.hpp:12 RangeFamily::exponential */

#define FBF_VARIANT_FUSED 0 /* one fused kernel (default)                        */
#define FBF_VARIANT_NAIVE 1 /* multi-kernel, HBM-resident planes (comparison)    */
/* ConvolutionBackend::recursive (spatial.hpp:98-112, recursive_gaussian.hpp):
 * the IIR Gaussian of the filter's sigma_s, fp64, whole images; like the
 * reference it applies to Gaussian windows with sigma_s >= 2 and falls back to
 * the direct (fused) path otherwise.  Through fbf_bilateral_fast_device and the
 * host entry points (not the prepare / filter_prepared split). */
#define FBF_VARIANT_RECURSIVE 2

/* Where the pixels are.  The global image is width x height.  A buffer holds
 * rows [src_row0, src_row0 + src_rows) of each of `batch` images (row strips
 * for multi-GPU sharding carry their W halo rows); rows [out_row0, out_row0 +
 * out_rows) are produced.  Pitches / strides are in elements. */
typedef struct fbf_geometry {
  int width, height;
  int batch;
  int src_row0, src_rows;
  int out_row0, out_rows;
  long long src_pitch, dst_pitch;
  long long src_bstride, dst_bstride;
} fbf_geometry;

/* SpatialKernel (spatial.hpp:22-33) + FourierKernelApprox (kernel_approx.hpp:19-44). */
typedef struct fbf_filter {
  int kind;               /* FBF_SPATIAL_*                                  */
  int radius;             /* W                                              */
  const double* profile;  /* 2W+1 normalised taps (host memory)             */
  double w0;              /* centre weight profile[W]^2                     */
  int N;                  /* highest harmonic                               */
  const double* d;        /* d_0..d_N (host memory)                         */
  double omega;           /* pi / T                                         */
  double max_pointwise_error; /* epsilon of the fit                         */
  int check_epsilon;      /* 1: enforce eps < w0 like bilateral.hpp:114-118 */
  double sigma_s;         /* spatial sigma (FBF_VARIANT_RECURSIVE); 0 if unknown */
} fbf_filter;

const char* fbf_last_error(void);
int fbf_version(void);

/* Fills g for a whole single image (or a batch of contiguous images). */
void fbf_geometry_whole(fbf_geometry* g, int width, int height, int batch);

/* Device workspace needed by fbf_bilateral_fast_device for spatial radius W (bytes). */
size_t fbf_workspace_bytes(const fbf_geometry* g, int radius, int variant);

/* Asynchronous, device-resident: src/dst/workspace are device pointers,
 * `stream` a cudaStream_t (NULL = legacy default).  d_bad (device, may be
 * NULL) receives atomicMin of the first collapsed-denominator linear index
 * (b*H*W + y*W + x); the caller initialises it to ~0ULL. */
int fbf_bilateral_fast_device(const fbf_geometry* g, const fbf_filter* f, const float* src,
                              float* dst, void* workspace, size_t workspace_bytes,
                              unsigned long long* d_bad, int variant, void* stream);

/* The two stages of fbf_bilateral_fast_device, for callers that time or
 * overlap them separately: (1) the per-pixel base phase u = round(f' omega/2pi
 * 2^32) and f' = f - 128 into the workspace; (2) the filter proper. */
int fbf_prepare_device(const fbf_geometry* g, const fbf_filter* f, const float* src,
                       void* workspace, size_t workspace_bytes, int variant, void* stream);
int fbf_filter_prepared_device(const fbf_geometry* g, const fbf_filter* f, float* dst,
                               void* workspace, size_t workspace_bytes,
                               unsigned long long* d_bad, int variant, void* stream);
/* Harmonic groups (CTA groups splitting the harmonics, each with its own
 * (Q, P) plane) the fused path uses for this geometry, radius and order N.
 * Every harmonic term is rounded once to a fixed-point grid and summed as an
 * integer, so the result is the same bits for any group count, strip or
 * batch partition, pipeline chunking or GPU split. */
int fbf_harmonic_groups(const fbf_geometry* g, int radius, int N);
/* Kernel launches one fbf_bilateral_fast_device call makes. */
int fbf_launches_per_call(const fbf_geometry* g, const fbf_filter* f, int variant);

/* Harmonic split (SURVEY.md §8(e) optional mode): the partial numerator and
 * denominator sums over harmonics [n_lo, n_hi) into pq_out, a dense device
 * array of (Q, P) fp64 pairs (batch x out_rows x width), after
 * fbf_prepare_device on the same workspace.  The values are exact multiples of
 * the call's fixed-point grid, so partial planes of disjoint harmonic ranges
 * sum exactly in any order (e.g. an NCCL fp64 all-reduce) to the bits of a
 * single-GPU call; fbf_finish_device then divides (with the reference's
 * collapse check) into dst. */
int fbf_partial_sums_device(const fbf_geometry* g, const fbf_filter* f, int n_lo, int n_hi,
                            double* pq_out, void* workspace, size_t workspace_bytes, int variant,
                            void* stream);
int fbf_finish_device(const fbf_geometry* g, const fbf_filter* f, const double* pq, float* dst,
                      unsigned long long* d_bad, void* stream);

/* Synchronous, host buffers (fp32): H2D, filter, D2H, pipelined in chunks
 * on two streams from 1 Mpixel.  On FBF_EANOMALY *bad_index holds the first
 * offending index. */
int fbf_bilateral_fast_host(const fbf_geometry* g, const fbf_filter* f, const float* src,
                            float* dst, int variant, long long* bad_index);

/* The host entry points keep one context per calling thread and device
 * (streams, a grow-only device buffer, pinned staging, a cached graph); this
 * frees the calling thread's (they are also freed when the thread exits). */
void fbf_release_host_buffers(void);

/* Same on fp64 host buffers (the reference Image stores doubles): the
 * double <-> float conversions run on a host thread pool into pinned staging,
 * overlapped chunk by chunk with the GPU pipeline. */
int fbf_bilateral_fast_host_f64(const fbf_geometry* g, const fbf_filter* f, const double* src,
                                double* dst, int variant, long long* bad_index);

/* One call over several GPUs of the box (devices[0..ndevices-1]), one host
 * worker thread per device: a batch is split by whole images, a single image
 * by row strips (16-row aligned cuts, each strip with its W halo rows; mirror
 * padding only at the global edges).  No exchange between devices; the result
 * equals the single-device call bit for bit. */
int fbf_bilateral_fast_host_multi(const fbf_geometry* g, const fbf_filter* f, const float* src,
                                  float* dst, int variant, long long* bad_index,
                                  const int* devices, int ndevices);
int fbf_bilateral_fast_host_multi_f64(const fbf_geometry* g, const fbf_filter* f,
                                      const double* src, double* dst, int variant,
                                      long long* bad_index, const int* devices, int ndevices);

/* convolve (spatial.hpp:98-112), direct backend: out(i) = sum_j profile[j+W]
 * in(i-j) along rows then columns, mirror boundaries, any radius.  Device
 * entry points in fp32 and fp64 (workspace: fbf_convolve_workspace_bytes);
 * the host entry is fp64 on the device, in the reference's summation order
 * (bit-identical to the reference). */
size_t fbf_convolve_workspace_bytes(int width, int height, int radius);
int fbf_convolve_device(int width, int height, const double* profile, int radius,
                        const float* src, float* dst, void* workspace, size_t workspace_bytes,
                        void* stream);
int fbf_convolve_device_f64(int width, int height, const double* profile, int radius,
                            const double* src, double* dst, void* workspace,
                            size_t workspace_bytes, void* stream);
int fbf_convolve_host_f64(int width, int height, const double* profile, int radius,
                          const double* src, double* dst);
/* convolve with the recursive backend: the IIR Gaussian of sigma (fp64; the
 * caller applies the reference's rule: Gaussian windows with sigma >= 2). */
int fbf_convolve_recursive_host_f64(int width, int height, double sigma, const double* src, double* dst);

/* bilateral_exact (bilateral.hpp:78-102) on the device in fp64: the O(W^2)
 * brute-force filter, for checking the paper's bound at full image sizes.
 * src: fp32 rows [src_row0, src_row0+src_rows) (dense, pitch = width);
 * dst: fp64 rows [out_row0, out_row0+out_rows); batch must be 1. */
int fbf_bilateral_exact_device(const fbf_geometry* g, const double* profile, int radius, int family,
                               double sigma_r, const float* src, double* dst, void* stream);

/* bilateral_exact of a whole fp64 host image, Gaussian or exponential range
 * kernel (the C++ API's bilateral_exact for those families; radius <= 64). */
int fbf_bilateral_exact_host_f64(int width, int height, const double* profile, int radius, int family,
                                 double sigma_r, const double* src, double* dst);

/* local_dynamic_range (bilateral.hpp:21-74) on the device, fp64 (exact):
 * *T = ceil(max over pixels of windowed max - windowed min). */
int fbf_local_dynamic_range_host_f64(const double* img, int width, int height, int W, int* T);

/* Host-side pieces of the path (stay on the CPU, as in the reference). */
int fbf_spatial_gaussian(double sigma_s, double* profile, int* radius, double* w0);
int fbf_spatial_box(int radius, double* profile, double* w0);
double fbf_range_eval(int family, double sigma_r, double t);
int fbf_fit_fixed(int family, double sigma_r, int T, int N, double* d, double* residual_norm,
                  double* max_pointwise_error);
int fbf_progressive_fit(int family, double sigma_r, int T, double epsilon, double* d, int* N,
                        double* residual_norm, double* max_pointwise_error);
double fbf_error_bound(int T, double epsilon, double w0);

/* Seeded synthetic image generator for the BASELINE configs (DESIGN.md
 * "inputs"): rows [row0, row0+rows) of a width x height image into out
 * (row-major, fp32), using nthreads host threads. */
int fbf_synth_image(unsigned long long seed, int width, int height, int rects, double noise_sigma,
                    int row0, int rows, float* out, int nthreads);

/* FP32 FMA-pipe peak of the current device, measured by a resident FFMA2
 * probe kernel: lane-ops per second and the SM clock it ran at. */
int fbf_probe_fma_peak(double* ops_per_s, double* sm_mhz, void* stream);

#ifdef __cplusplus
}
#endif
#endif
