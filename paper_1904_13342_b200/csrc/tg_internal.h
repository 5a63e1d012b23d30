// tg_internal.h — shared host-side plumbing of libtomograd_b200 (not part of the ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "tomograd_b200.h"

namespace tgb {

// A reference check() failure (tomograd::Error, core.hpp:19-26); the text is
// the reference's exact message.
struct RefError : std::runtime_error {
  explicit RefError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(bool cond, const char* msg) {
  if (!cond) throw RefError(msg);
}

void set_last_error(const std::string& msg);

// Translate exceptions into tg_status at the ABI edge.
template <typename Fn>
tg_status guarded(Fn&& fn) {
  try {
    fn();
    return TG_OK;
  } catch (const RefError& e) {
    set_last_error(e.what());
    return TG_ERROR;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return TG_ERROR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TG_ERROR;
  }
}

// ---- host geometry (host_geometry.cpp; bit-exact with the reference) -----
constexpr double kPi = 3.14159265358979323846;

void view_angles(uint64_t n, double range, double* out);
void cone_projection_matrix(double theta, double sid, double sdd, const tg_detector2d& det,
                            double* m);
void cone_set_matrices(uint64_t n, double sid, const double* in, double* mats, double* sources,
                       double* invs, double* angles);
void validate_volume(const tg_volume_spec& v);
double cone_fan_half_angle(const tg_cone_geometry& g);
double planar_fan_half_angle(const tg_planar_geometry& g);
double parker_delta(double range, double fan_half_angle);
double parker_weight(double beta, double gamma, double delta, double range);
void cosine_weights_cone(const tg_cone_geometry& g, double* out);
void parker_weights_cone(const tg_cone_geometry& g, double* out);
void ramlak_weights(uint64_t P, double spacing, double* out);
bool is_pow2(uint64_t n);
uint64_t next_pow2(uint64_t n);
void head_ellipsoids(double fov_half, double* out80);
void head_ellipses(double fov_half, double* out60);
double fov_half_extent(const tg_volume_spec& v);

// ---- instrumentation ------------------------------------------------------
void count_launch(uint64_t n = 1);

}  // namespace tgb
