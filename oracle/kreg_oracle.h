/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference CVO registration hot path
 * (/root/reference/proj/src: se3.cpp, kernels.cpp, hash_grid.cpp,
 * inner_product.cpp, reference.cpp, registration.cpp; include/kreg/detail/
 * reduce.hpp). It is the CPU checker the parity tests compare the CUDA path
 * against, and the "port" CPU baseline. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it (through liboracle.so).
 *
 * Pinned against: the compiled reference itself (oracle/_ref/libkreg_ref.so,
 * built from the reference sources by oracle/Makefile) and the golden
 * vectors under tests/golden/ generated from it (tests/golden/make_golden.py).
 *
 * POD descriptors are shared with the product ABI (include/kreg_b200.h).
 */
#ifndef KREG_ORACLE_H_
#define KREG_ORACLE_H_

#include "../include/kreg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ko_pairs ko_pairs;

const char* ko_last_error(void);

/* se3.cpp:48-76 */
int ko_se3_exp(const double xi[6], double T[12]);
/* se3.cpp:109-120 (re-orthonormalises when Gram drift > 1e-7, :115-118) */
void ko_se3_compose(const double a[12], const double b[12], double out[12]);
/* se3.cpp:122-127 */
void ko_se3_inverse(const double T[12], double out[12]);
/* kernels.cpp:18-53 */
double ko_feature_coefficient(const double* u, const double* v, const kreg_cloud_view* schema,
                              const kreg_kernel_params* params);
/* inner_product.cpp:37-95 (grid search) ; reference.cpp:9-37 when dense != 0 */
int ko_build_pairs(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                   const kreg_kernel_params* params, double cutoff_multiplier, double c_min,
                   int dense, ko_pairs** out, int64_t* n_pairs);
void ko_pairs_destroy(ko_pairs* p);
void ko_pairs_export(const ko_pairs* p, int64_t* offsets, int32_t* x_index, double* coeff);
/* inner_product.cpp:97-119 */
double ko_inner_product(const ko_pairs* p, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                        const double T[12], const kreg_kernel_params* params);
/* inner_product.cpp:121-152 ; out = {F, omega[3], v[3]} */
void ko_objective_and_gradient(const ko_pairs* p, const kreg_cloud_view* X,
                               const kreg_cloud_view* Z, const double T[12],
                               const kreg_kernel_params* params, double out[7]);
/* inner_product.cpp:238-246 */
void ko_directional_terms(const ko_pairs* p, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                          const double T[12], const double xi[6], const kreg_kernel_params* params, double out[3]);
double ko_max_point_displacement(const kreg_cloud_view* Z, const double built[12],
                                 const double now[12]);
/* point_cloud.cpp:69-87 */
double ko_diameter(const kreg_cloud_view* X);
/* registration.cpp:36-52 */
double ko_anneal_step(double lengthscale, const double* history, int n,
                      const kreg_registration_config* config);
/* registration.cpp:12-34 ; returns 0 or KREG_INVALID_ARGUMENT */
int ko_check_config(const kreg_registration_config* config);
/* registration.cpp:100-189 ; returns KREG_OK / KREG_NO_OVERLAP / KREG_INVALID_ARGUMENT */
int ko_register_clouds(const kreg_cloud_view* X, const kreg_cloud_view* Z,
                       const double initial[12], const kreg_kernel_params* params,
                       const kreg_registration_config* config, kreg_registration_result* result);
/* Replay log for the next ko_register_clouds calls on this process (NULL /
 * cap 0 disables): per iteration T (12), the pair list's build transform (12)
 * and the lengthscale. */
void ko_set_iteration_log(double* T, double* Tb, double* l, int cap);
/* image.cpp:144-155 integer rec601 luma (channels 1 or >= 3) */
void ko_to_gray(const uint8_t* rgb, int channels, int w, int h, uint8_t* gray);
/* selector.cpp:29-51 segment test (16-pixel circle, 9 contiguous, strict) */
int ko_is_corner(const uint8_t* gray, int w, int u, int v, double t);
/* selector.cpp:63-125: the budgeted selection; pixels (u, v) raster order,
 * capacity w*h pairs; returns the count, fills threshold / in_band / fallback */
long ko_select_points(const uint8_t* rgb, int channels, int w, int h, const uint8_t* valid,
                      const kreg_selector_config* sel, int32_t* pixels, double* threshold, int* in_band,
                      int* fallback);
/* projection.cpp:30-75: rows xyz (3) and features (3 + sem_ch), capacity w*h */
long ko_depth_rgb_to_cloud(const uint16_t* depth, const uint8_t* rgb, int channels, const float* sem, int sem_ch,
                           int w, int h, const kreg_camera_intrinsics* intr, const kreg_selector_config* sel,
                           double* xyz, double* feat, int* fallback, int* in_band);
/* rng.hpp:11-46 SplitMix64 helpers for fixtures */
uint64_t ko_splitmix_next(uint64_t* state);
uint64_t ko_splitmix_derive(uint64_t seed, uint64_t index);

#ifdef __cplusplus
}
#endif

#endif
