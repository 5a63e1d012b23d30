#pragma once

// Drop-in replacement for the reference toolkit's tomograd/projector.hpp
// (proj/include/tomograd/projector.hpp:169-313): the same six overloads,
// template signatures, shape checks and error text, running on a B200
// through the C ABI of libtomograd_b200.so (include/tomograd_b200.h).
//
// Use: put  -I<repo>/include/tomograd_b200  before the reference's include
// directory and link -ltomograd_b200.  Every reference header that includes
// "tomograd/projector.hpp" (graph.hpp, pipelines.hpp, cli.hpp) then calls the
// GPU operators unchanged.  The reference's own geometry / image headers are
// used as-is.  T = float goes straight through; T = double is converted at the
// host<->device copy (the device computes in fp32).
//
// Plans (device-resident geometry) are cached per geometry content, so the
// graph's repeated forward/backward calls do not rebuild them.

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "tomograd/core.hpp"
#include "tomograd/geometry.hpp"
#include "tomograd/image.hpp"
#include "tomograd_b200.h"

namespace tomograd {

namespace b200 {

inline void throw_if(tg_status s) {
  if (s != TG_OK) throw Error(tg_last_error());
}

inline int device() {
  static const int d = [] {
    const char* e = std::getenv("TOMOGRAD_B200_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return d;
}

inline tg_volume_spec to_c(const VolumeSpec& v) {
  tg_volume_spec c{};
  c.dims = uint32_t(v.shape.size());
  for (std::size_t a = 0; a < v.shape.size() && a < 3; ++a) {
    c.shape[a] = v.shape[a];
    c.spacing[a] = v.spacing[a];
    c.origin[a] = a < v.origin.size() ? v.origin[a] : 0.0;
  }
  return c;
}

// FNV-1a over the bytes that define a geometry
struct Hasher {
  uint64_t h = 1469598103934665603ull;
  void add(const void* p, std::size_t n) {
    auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
  template <typename T>
  void add(const std::vector<T>& v) {
    add(v.data(), v.size() * sizeof(T));
  }
  void add(double d) { add(&d, sizeof d); }
};

template <typename Plan, tg_status (*Destroy)(Plan*)>
struct PlanCache {
  std::mutex mu;
  std::unordered_map<uint64_t, std::shared_ptr<Plan>> plans;
  template <typename Make>
  std::shared_ptr<Plan> get(uint64_t key, Make make) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = plans.find(key);
    if (it != plans.end()) return it->second;
    Plan* p = nullptr;
    throw_if(make(&p));
    std::shared_ptr<Plan> sp(p, [](Plan* q) { Destroy(q); });
    if (plans.size() > 64) plans.clear();
    plans.emplace(key, sp);
    return sp;
  }
};

inline PlanCache<tg_cone_plan, tg_cone_plan_destroy>& cone_cache() {
  static PlanCache<tg_cone_plan, tg_cone_plan_destroy> c;
  return c;
}
inline PlanCache<tg_planar_plan, tg_planar_plan_destroy>& planar_cache() {
  static PlanCache<tg_planar_plan, tg_planar_plan_destroy> c;
  return c;
}

inline std::shared_ptr<tg_cone_plan> cone_plan(const ConeGeometry& g) {
  Hasher h;
  h.add(g.volume.shape);
  h.add(g.volume.spacing);
  h.add(g.volume.origin);
  h.add(&g.detector, sizeof g.detector);
  h.add(g.angular_range);
  h.add(g.sid);
  h.add(g.sdd);
  for (const auto& m : g.matrices) h.add(m.m.data(), sizeof(double) * 12);
  h.add(g.angles);
  return cone_cache().get(h.h, [&](tg_cone_plan** out) {
    std::vector<double> mats, src, inv;
    for (const auto& m : g.matrices) mats.insert(mats.end(), m.m.begin(), m.m.end());
    for (const auto& s : g.sources) src.insert(src.end(), {s.x, s.y, s.z});
    for (const auto& b : g.inv_blocks) inv.insert(inv.end(), b.m.begin(), b.m.end());
    tg_cone_geometry c{to_c(g.volume),
                       {g.detector.n_u, g.detector.n_v, g.detector.spacing_u, g.detector.spacing_v,
                        g.detector.origin_u, g.detector.origin_v},
                       g.n_projections, g.angular_range, g.sid, g.sdd, mats.data(), src.data(),
                       inv.data(), g.angles.data()};
    return tg_cone_plan_create(&c, device(), out);
  });
}

template <typename G>
inline std::shared_ptr<tg_planar_plan> planar_plan(const G& g, double sid, double sdd) {
  Hasher h;
  h.add(g.volume.shape);
  h.add(g.volume.spacing);
  h.add(g.volume.origin);
  h.add(&g.detector, sizeof g.detector);
  h.add(sid);
  h.add(sdd);
  for (const auto& r : g.rays) h.add(&r, sizeof r);
  return planar_cache().get(h.h, [&](tg_planar_plan** out) {
    std::vector<double> rays;
    for (const auto& r : g.rays) rays.insert(rays.end(), {r.x, r.y});
    tg_planar_geometry c{to_c(g.volume), {g.detector.n_bins, g.detector.spacing, g.detector.origin},
                         g.n_projections, g.angular_range, sid, sdd, rays.data(), g.angles.data()};
    return tg_planar_plan_create(&c, device(), out);
  });
}

// fp32 views of T data (no copy for T = float)
template <typename T>
struct F32In {
  std::vector<float> buf;
  const float* p;
  explicit F32In(const std::vector<T>& v) {
    if constexpr (std::is_same_v<T, float>) {
      p = v.data();
    } else {
      buf.assign(v.begin(), v.end());
      p = buf.data();
    }
  }
};

template <typename T>
struct F32Out {
  std::vector<T>& dst;
  std::vector<float> buf;
  float* p;
  explicit F32Out(std::vector<T>& v) : dst(v) {
    if constexpr (std::is_same_v<T, float>) {
      p = v.data();
    } else {
      buf.resize(v.size());
      p = buf.data();
    }
  }
  void commit() {
    if constexpr (!std::is_same_v<T, float>)
      for (std::size_t i = 0; i < buf.size(); ++i) dst[i] = T(buf[i]);
  }
};

}  // namespace b200

namespace detail {

// projector.hpp:154-165
inline void check_volume_match(const VolumeSpec& a, const VolumeSpec& b) {
  check(a.shape == b.shape && a.spacing == b.spacing && a.origin == b.origin,
        "volume does not match the geometry's volume spec");
}

template <typename T>
inline void check_sino_match(const Sinogram<T>& s, std::size_t n_proj, std::size_t n_bins) {
  check(!s.is_cone() && s.n_projections == n_proj && s.detector1d.n_bins == n_bins,
        "sinogram shape does not match the geometry");
}

}  // namespace detail

// --- parallel beam: projector.hpp:171-208 ----------------------------------

template <typename T>
Sinogram<T> forward_project(const Image<T>& img, const ParallelGeometry& geo) {
  detail::check_volume_match(img.spec, geo.volume);
  auto sino = Sinogram<T>::planar(geo.n_projections, geo.detector);
  auto plan = b200::planar_plan(geo, 0.0, 0.0);
  b200::F32In<T> in(img.data);
  b200::F32Out<T> out(sino.data);
  b200::throw_if(tg_planar_forward_host(plan.get(), in.p, out.p));
  out.commit();
  return sino;
}

template <typename T>
Image<T> back_project(const Sinogram<T>& sino, const ParallelGeometry& geo) {
  detail::check_sino_match(sino, geo.n_projections, geo.detector.n_bins);
  Image<T> img(geo.volume);
  auto plan = b200::planar_plan(geo, 0.0, 0.0);
  b200::F32In<T> in(sino.data);
  b200::F32Out<T> out(img.data);
  b200::throw_if(tg_planar_backproject_host(plan.get(), in.p, out.p));
  out.commit();
  return img;
}

// --- fan beam: projector.hpp:212-260 ---------------------------------------

template <typename T>
Sinogram<T> forward_project(const Image<T>& img, const FanGeometry& geo) {
  detail::check_volume_match(img.spec, geo.volume);
  auto sino = Sinogram<T>::planar(geo.n_projections, geo.detector);
  auto plan = b200::planar_plan(geo, geo.sid, geo.sdd);
  b200::F32In<T> in(img.data);
  b200::F32Out<T> out(sino.data);
  b200::throw_if(tg_planar_forward_host(plan.get(), in.p, out.p));
  out.commit();
  return sino;
}

template <typename T>
Image<T> back_project(const Sinogram<T>& sino, const FanGeometry& geo) {
  detail::check_sino_match(sino, geo.n_projections, geo.detector.n_bins);
  Image<T> img(geo.volume);
  auto plan = b200::planar_plan(geo, geo.sid, geo.sdd);
  b200::F32In<T> in(sino.data);
  b200::F32Out<T> out(img.data);
  b200::throw_if(tg_planar_backproject_host(plan.get(), in.p, out.p));
  out.commit();
  return img;
}

// --- cone beam: projector.hpp:264-313 ---------------------------------------

template <typename T>
Sinogram<T> forward_project(const Image<T>& img, const ConeGeometry& geo) {
  detail::check_volume_match(img.spec, geo.volume);
  auto sino = Sinogram<T>::cone_beam(geo.n_projections, geo.detector);
  auto plan = b200::cone_plan(geo);
  b200::F32In<T> in(img.data);
  b200::F32Out<T> out(sino.data);
  b200::throw_if(tg_cone_forward_host(plan.get(), in.p, out.p));
  out.commit();
  return sino;
}

template <typename T>
Image<T> back_project(const Sinogram<T>& sino, const ConeGeometry& geo) {
  check(sino.is_cone() && sino.n_projections == geo.n_projections &&
            sino.detector2d.n_u == geo.detector.n_u && sino.detector2d.n_v == geo.detector.n_v,
        "sinogram shape does not match the geometry");
  Image<T> img(geo.volume);
  auto plan = b200::cone_plan(geo);
  b200::F32In<T> in(sino.data);
  b200::F32Out<T> out(img.data);
  b200::throw_if(tg_cone_backproject_host(plan.get(), in.p, out.p));
  out.commit();
  return img;
}

namespace b200 {

// pipelines.hpp:73-84 fdk_reconstruct with the weights, Ram-Lak filter and
// back-projection all on the device (one call; the reference's version runs
// weights and filter serially on the host).
template <typename T>
Image<T> fdk_reconstruct(const Sinogram<T>& sino, const ConeGeometry& geo, bool use_parker = true) {
  check(sino.is_cone() && sino.n_projections == geo.n_projections &&
            sino.detector2d.n_u == geo.detector.n_u && sino.detector2d.n_v == geo.detector.n_v,
        "sinogram shape does not match the geometry");
  Image<T> img(geo.volume);
  auto plan = cone_plan(geo);
  F32In<T> in(sino.data);
  F32Out<T> out(img.data);
  throw_if(tg_cone_fdk_host(plan.get(), in.p, out.p, use_parker ? 1 : 0));
  out.commit();
  return img;
}

// pipelines.hpp:273-299 tv_reconstruct (x -> forward_project -> l2_loss(., p)
// + tv_lambda * tv_loss(x), plain gradient descent from zero) with the whole
// loop device resident: projections, l2 residual, TV subgradient and the
// descent step never leave HBM; only the loss history returns.  Any
// geometry type (the reference's graph nodes take all three).  The config
// type is the caller's ExperimentConfig (learning_rate, iterations,
// tv_lambda), so this header stays independent of pipelines.hpp.
template <typename T, typename Geo, typename Cfg>
std::pair<Image<T>, std::vector<double>> tv_reconstruct(const Sinogram<T>& sino, const Geo& geo,
                                                        const Cfg& cfg) {
  Image<T> img(geo.volume);
  std::vector<double> hist(cfg.iterations + 1);
  F32In<T> in(sino.data);
  std::vector<float> x(img.data.size(), 0.0f);
  const std::size_t nvox = x.size();
  if constexpr (std::is_same_v<Geo, ConeGeometry>) {
    check(sino.is_cone() && sino.n_projections == geo.n_projections &&
              sino.detector2d.n_u == geo.detector.n_u && sino.detector2d.n_v == geo.detector.n_v,
          "sinogram shape does not match the geometry");
    throw_if(tg_cone_tv_reconstruct_host(cone_plan(geo).get(), in.p, x.data(), cfg.iterations,
                                         cfg.learning_rate, cfg.tv_lambda, hist.data()));
  } else {
    check(!sino.is_cone() && sino.n_projections == geo.n_projections &&
              sino.detector1d.n_bins == geo.detector.n_bins,
          "sinogram shape does not match the geometry");
    double sid = 0.0, sdd = 0.0;
    if constexpr (std::is_same_v<Geo, FanGeometry>) {
      sid = geo.sid;
      sdd = geo.sdd;
    }
    throw_if(tg_planar_tv_reconstruct_host(planar_plan(geo, sid, sdd).get(), in.p, x.data(),
                                           cfg.iterations, cfg.learning_rate, cfg.tv_lambda,
                                           hist.data()));
  }
  for (std::size_t i = 0; i < nvox; ++i) img.data[i] = T(x[i]);
  return {std::move(img), std::move(hist)};
}

// pipelines.hpp:211-259 (experiment_learn_filter's graph loop) device
// resident: frequency weights K start at init_weights (the ramp) and descend
// on |pi/n BP(fourier_filter(p, K)) - target|^2 (target: the Ram-Lak FBP of p);
// every step's filter, projections, gradients and update stay in HBM, one
// step captured as a CUDA graph.  Returns the learned weights, the loss and
// distance (|K - ramlak| / |init - ramlak|) histories and the reconstruction.
template <typename T>
struct LearnFilterResult {
  std::vector<double> loss_history, distance_history, learned_weights;
  Image<T> reconstruction;
};

template <typename T>
LearnFilterResult<T> learn_filter(const Sinogram<T>& sino, const ParallelGeometry& geo,
                                  const Image<T>& target, const std::vector<double>& init_weights,
                                  const std::vector<double>& ramlak_weights, double learning_rate,
                                  std::size_t iterations) {
  check(!sino.is_cone() && sino.n_projections == geo.n_projections &&
            sino.detector1d.n_bins == geo.detector.n_bins,
        "sinogram shape does not match the geometry");
  check(init_weights.size() == ramlak_weights.size(),
        "filter window is inconsistent with its weight vector");
  LearnFilterResult<T> r;
  r.reconstruction = Image<T>(geo.volume);
  F32In<T> in(sino.data), tgt(target.data);
  std::vector<float> k(init_weights.begin(), init_weights.end());
  std::vector<float> rec(r.reconstruction.data.size());
  r.loss_history.resize(iterations + 1);
  r.distance_history.resize(iterations + 1);
  throw_if(tg_planar_learn_filter_host(planar_plan(geo, 0.0, 0.0).get(), in.p, tgt.p, k.data(),
                                       k.size(), init_weights.data(), ramlak_weights.data(),
                                       learning_rate, iterations, r.loss_history.data(),
                                       r.distance_history.data(), rec.data()));
  r.learned_weights.assign(k.begin(), k.end());
  for (std::size_t i = 0; i < rec.size(); ++i) r.reconstruction.data[i] = T(rec[i]);
  return r;
}

}  // namespace b200
}  // namespace tomograd
