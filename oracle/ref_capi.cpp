// ref_capi.cpp — CPU ORACLE glue (TEST INFRASTRUCTURE ONLY).
//
// Compiles the UNMODIFIED reference toolkit headers (found through
// -I$(TOMOGRAD_REF_INCLUDE), default /root/reference/proj/include) into
// oracle/_ref/libtomograd_ref.so and exposes its projector / FDK path through
// a C ABI that uses the same POD structs as the C restatement (tg_oracle.h).
// Nothing here re-implements an algorithm: every call goes to the
// reference's own functions.  Used only to pin the restatement (tests/) and
// as bench.py's "reference" CPU arm.
#include <cmath>
#include <cstring>
#include <numbers>
#include <exception>
#include <string>
#include <vector>

#include "tg_oracle.h"
#include "tomograd/filtering.hpp"
#include "tomograd/geometry.hpp"
#include "tomograd/graph.hpp"
#include "tomograd/image.hpp"
#include "tomograd/phantom.hpp"
#include "tomograd/pipelines.hpp"
#include "tomograd/projector.hpp"

using namespace tomograd;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

VolumeSpec to_spec(const or_volume& v) {
  VolumeSpec s;
  for (uint32_t a = 0; a < v.dims; ++a) {
    s.shape.push_back(std::size_t(v.shape[a]));
    s.spacing.push_back(v.spacing[a]);
    s.origin.push_back(v.origin[a]);
  }
  return s;
}

Detector1D to_det(const or_det1& d) { return {std::size_t(d.n_bins), d.spacing, d.origin}; }
Detector2D to_det(const or_det2& d) {
  return {std::size_t(d.n_u), std::size_t(d.n_v), d.spacing_u, d.spacing_v, d.origin_u, d.origin_v};
}

// Planar geometry: circular (rays == nullptr) through the reference factories,
// otherwise with explicit rays (ParallelGeometry::set_custom_rays semantics
// are not needed: rays are stored as given, angles as given).
ParallelGeometry to_parallel(const or_planar& g) {
  auto geo = make_parallel(to_spec(g.vol), to_det(g.det), std::size_t(g.n_proj), g.range);
  return geo;
}
FanGeometry to_fan(const or_planar& g) {
  return make_fan(to_spec(g.vol), to_det(g.det), std::size_t(g.n_proj), g.range, g.sid, g.sdd);
}

// Cone geometry through the reference's own setup: circular via make_cone,
// explicit (already normalised) matrices via make_cone_from_matrices.
ConeGeometry to_cone(const or_cone& g, bool circular) {
  if (circular)
    return make_cone(to_spec(g.vol), to_det(g.det), std::size_t(g.n_proj), g.range, g.sid, g.sdd);
  std::vector<Mat34> mats(g.n_proj);
  for (std::size_t i = 0; i < g.n_proj; ++i)
    for (int k = 0; k < 12; ++k) mats[i].m[std::size_t(k)] = g.mats[12 * i + std::size_t(k)];
  return make_cone_from_matrices(to_spec(g.vol), to_det(g.det), g.range, g.sid, g.sdd, mats);
}

template <typename T>
Image<T> make_image(const VolumeSpec& s, const T* data) {
  Image<T> img(s);
  std::memcpy(img.data.data(), data, sizeof(T) * img.data.size());
  return img;
}

// pipelines.hpp:276-298 tv_reconstruct, instantiated for any geometry through
// the reference's own Graph (its nodes take every geometry type,
// graph.hpp:117-135); for ParallelGeometry the reference function itself is
// called (ref_tv_reconstruct_parallel).
template <typename Geo>
std::vector<double> tv_graph(const Sinogram<>& sino, const Geo& geo, const ExperimentConfig& cfg,
                             std::vector<double>& x_out) {
  Graph g;
  const NodeId x = g.parameter(Tensor<>(geo.volume.shape), /*trainable=*/true);
  const NodeId p = g.input(sino.shape());
  const NodeId fp = g.forward_project(x, geo);
  const NodeId data_term = g.l2_loss(fp, p);
  const NodeId loss = g.add(data_term, g.scale(g.tv_loss(x), cfg.tv_lambda));
  std::vector<double> history;
  const std::map<NodeId, Tensor<>> feeds{{p, sino.tensor()}};
  for (std::size_t it = 0; it < cfg.iterations; ++it) {
    g.forward(feeds);
    history.push_back(g.value(loss).scalar_value());
    check_converging(history.back(), it);
    const auto grads = g.backward(loss);
    gradient_descent_step(g, grads, cfg.learning_rate);
  }
  g.forward(feeds);
  history.push_back(g.value(loss).scalar_value());
  check_converging(history.back(), cfg.iterations);
  x_out = g.node(x).value.data;
  return history;
}

// pipelines.hpp:211-259 (experiment_learn_filter's graph and loop) on a
// given sinogram: the same nodes, feeds, record and descent order, so the
// device graph can be compared on an identical fp32 input.  Pinned against
// the reference function itself by ref_experiment_learn_filter (tests).
void learn_filter_graph(const Sinogram<>& sino, const ParallelGeometry& geo, std::size_t window,
                        double lr, std::size_t iterations, std::vector<double>& loss_h,
                        std::vector<double>& dist_h, std::vector<double>& weights,
                        std::vector<double>& recon_out) {
  const Filter1D ramp = ramp_filter(geo.detector.n_bins, geo.detector.spacing, window);
  const Filter1D ramlak = ramlak_filter(geo.detector.n_bins, geo.detector.spacing, window);
  const std::size_t padded = ramp.padded_n;
  double gap = 0.0;
  for (std::size_t k = 0; k < padded; ++k) {
    const double d = ramp.weights[k] - ramlak.weights[k];
    gap += d * d;
  }
  gap = std::sqrt(gap);
  Image<> reference = fbp_reconstruct(sino, geo, ramlak);
  Graph g;
  const NodeId p = g.input(sino.shape());
  const NodeId K = g.parameter(Tensor<>({padded}, ramp.weights), true);
  const NodeId target = g.parameter(reference.tensor(), false);
  const NodeId filtered = g.fourier_filter(p, K, padded);
  const NodeId bp = g.backproject(filtered, geo);
  const NodeId recon = g.scale(bp, std::numbers::pi / double(geo.n_projections));
  const NodeId loss = g.l2_loss(recon, target);
  const std::map<NodeId, Tensor<>> feeds{{p, sino.tensor()}};
  auto record = [&] {
    loss_h.push_back(g.value(loss).scalar_value());
    double d2 = 0.0;
    const auto& w = g.node(K).value.data;
    for (std::size_t k = 0; k < padded; ++k) {
      const double d = w[k] - ramlak.weights[k];
      d2 += d * d;
    }
    dist_h.push_back(gap > 0.0 ? std::sqrt(d2) / gap : 0.0);
  };
  for (std::size_t it = 0; it < iterations; ++it) {
    g.forward(feeds);
    record();
    const auto grads = g.backward(loss);
    gradient_descent_step(g, grads, lr);
  }
  g.forward(feeds);
  record();
  weights = g.node(K).value.data;
  recon_out = g.value(recon).data;
}

}  // namespace

extern "C" {

// the graph of experiment_learn_filter on a given sinogram (see above)
int ref_learn_filter_graph(const or_planar* gp, const double* sino, uint64_t window, double lr,
                           uint64_t iterations, double* loss_h, double* dist_h, double* weights,
                           double* recon) {
  return guard([&] {
    const auto geo = to_parallel(*gp);
    auto s = Sinogram<>::planar(geo.n_projections, geo.detector);
    std::memcpy(s.data.data(), sino, sizeof(double) * s.data.size());
    std::vector<double> l, d, w, r;
    learn_filter_graph(s, geo, std::size_t(window), lr, std::size_t(iterations), l, d, w, r);
    std::memcpy(loss_h, l.data(), sizeof(double) * l.size());
    std::memcpy(dist_h, d.data(), sizeof(double) * d.size());
    std::memcpy(weights, w.data(), sizeof(double) * w.size());
    std::memcpy(recon, r.data(), sizeof(double) * r.size());
  });
}

// pipelines.hpp:196-261 experiment_learn_filter itself (phantom by name)
int ref_experiment_learn_filter(const or_planar* gp, const char* phantom, double noise,
                                uint64_t seed, uint64_t window, double lr, uint64_t iterations,
                                double* loss_h, double* dist_h, double* weights, double* recon,
                                uint64_t* padded_out) {
  return guard([&] {
    const auto geo = to_parallel(*gp);
    ExperimentConfig cfg;
    cfg.phantom = phantom;
    cfg.noise_relative_std = noise;
    cfg.seed = seed;
    cfg.filter_window = std::size_t(window);
    cfg.learning_rate = lr;
    cfg.iterations = std::size_t(iterations);
    auto r = experiment_learn_filter(geo, cfg);
    std::memcpy(loss_h, r.loss_history.data(), sizeof(double) * r.loss_history.size());
    std::memcpy(dist_h, r.distance_history.data(), sizeof(double) * r.distance_history.size());
    std::memcpy(weights, r.learned_weights.data(), sizeof(double) * r.learned_weights.size());
    std::memcpy(recon, r.reconstruction.data.data(), sizeof(double) * r.reconstruction.data.size());
    *padded_out = r.ramp_init.padded_n;
  });
}

// One forward + backward of a graph exercising the node kinds that
// experiment_learn_filter does not:
//   loss = l2(multiply_weights(forward_project(x), w), p) + scale(tv(x), lambda)
// Outputs the loss and the gradients of x (image) and w (row weights, n_bins).
int ref_graph_probe(const or_planar* gp, int fan, const double* x0, const double* w0,
                    const double* sino, double lambda, double* loss, double* gx, double* gw) {
  return guard([&] {
    Graph g;
    auto run = [&](const auto& geo) {
      std::size_t nvox = 1;
      for (auto d : geo.volume.shape) nvox *= d;
      const NodeId x =
          g.parameter(Tensor<>(geo.volume.shape, std::vector<double>(x0, x0 + nvox)), true);
      const NodeId w = g.parameter(Tensor<>({geo.detector.n_bins},
                                            std::vector<double>(w0, w0 + geo.detector.n_bins)),
                                   true);
      auto s = Sinogram<>::planar(geo.n_projections, geo.detector);
      const NodeId p = g.input(s.shape());
      std::memcpy(s.data.data(), sino, sizeof(double) * s.data.size());
      const NodeId fp = g.forward_project(x, geo);
      const NodeId mw = g.multiply_weights(fp, w);
      const NodeId data_term = g.l2_loss(mw, p);
      const NodeId l = g.add(data_term, g.scale(g.tv_loss(x), lambda));
      g.forward({{p, s.tensor()}});
      *loss = g.value(l).scalar_value();
      auto grads = g.backward(l);
      std::memcpy(gx, grads[x].data.data(), sizeof(double) * grads[x].data.size());
      std::memcpy(gw, grads[w].data.data(), sizeof(double) * grads[w].data.size());
    };
    if (fan)
      run(to_fan(*gp));
    else
      run(to_parallel(*gp));
  });
}

int ref_tv_reconstruct_parallel(const or_planar* g, const double* sino, double* x,
                                uint64_t iterations, double lr, double lambda, double* hist) {
  return guard([&] {
    const auto geo = to_parallel(*g);
    auto s = Sinogram<>::planar(geo.n_projections, geo.detector);
    std::memcpy(s.data.data(), sino, sizeof(double) * s.data.size());
    ExperimentConfig cfg;
    cfg.learning_rate = lr;
    cfg.iterations = std::size_t(iterations);
    cfg.tv_lambda = lambda;
    auto [rec, h] = tv_reconstruct(s, geo, cfg);
    std::memcpy(x, rec.data.data(), sizeof(double) * rec.data.size());
    std::memcpy(hist, h.data(), sizeof(double) * h.size());
  });
}

int ref_tv_reconstruct_fan(const or_planar* g, const double* sino, double* x, uint64_t iterations,
                           double lr, double lambda, double* hist) {
  return guard([&] {
    const auto geo = to_fan(*g);
    auto s = Sinogram<>::planar(geo.n_projections, geo.detector);
    std::memcpy(s.data.data(), sino, sizeof(double) * s.data.size());
    ExperimentConfig cfg;
    cfg.learning_rate = lr;
    cfg.iterations = std::size_t(iterations);
    cfg.tv_lambda = lambda;
    std::vector<double> xv;
    auto h = tv_graph(s, geo, cfg, xv);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    std::memcpy(hist, h.data(), sizeof(double) * h.size());
  });
}

int ref_tv_reconstruct_cone(const or_cone* g, int circular, const double* sino, double* x,
                            uint64_t iterations, double lr, double lambda, double* hist) {
  return guard([&] {
    const auto geo = to_cone(*g, circular != 0);
    auto s = Sinogram<>::cone_beam(geo.n_projections, geo.detector);
    std::memcpy(s.data.data(), sino, sizeof(double) * s.data.size());
    ExperimentConfig cfg;
    cfg.learning_rate = lr;
    cfg.iterations = std::size_t(iterations);
    cfg.tv_lambda = lambda;
    std::vector<double> xv;
    auto h = tv_graph(s, geo, cfg, xv);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    std::memcpy(hist, h.data(), sizeof(double) * h.size());
  });
}

// pipelines.hpp:119-132 on a planar sinogram of n values (the stream depends
// only on the flat data order)
int ref_add_gaussian_noise_f64(const double* in, double* out, uint64_t n, double rel,
                               uint64_t seed) {
  return guard([&] {
    Detector1D d{std::size_t(n), 1.0, 0.0};
    auto s = Sinogram<double>::planar(1, d);
    std::memcpy(s.data.data(), in, sizeof(double) * n);
    auto o = add_gaussian_noise(s, rel, seed);
    std::memcpy(out, o.data.data(), sizeof(double) * n);
  });
}

int ref_add_gaussian_noise_f32(const float* in, float* out, uint64_t n, double rel, uint64_t seed) {
  return guard([&] {
    Detector1D d{std::size_t(n), 1.0, 0.0};
    auto s = Sinogram<float>::planar(1, d);
    std::memcpy(s.data.data(), in, sizeof(float) * n);
    auto o = add_gaussian_noise(s, rel, seed);
    std::memcpy(out, o.data.data(), sizeof(float) * n);
  });
}


const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(int n) { set_num_threads(unsigned(n < 1 ? 1 : n)); }
int ref_num_threads(void) { return int(num_threads()); }

int ref_view_angles(uint64_t n, double range, double* out) {
  return guard([&] {
    auto a = view_angles(std::size_t(n), range);
    std::memcpy(out, a.data(), sizeof(double) * a.size());
  });
}

int ref_make_cone(const or_volume* vol, const or_det2* det, uint64_t n, double range, double sid,
                  double sdd, double* mats, double* sources, double* invs, double* angles) {
  return guard([&] {
    auto g = make_cone(to_spec(*vol), to_det(*det), std::size_t(n), range, sid, sdd);
    for (std::size_t i = 0; i < n; ++i) {
      std::memcpy(mats + 12 * i, g.matrices[i].m.data(), 12 * sizeof(double));
      std::memcpy(invs + 9 * i, g.inv_blocks[i].m.data(), 9 * sizeof(double));
      sources[3 * i] = g.sources[i].x;
      sources[3 * i + 1] = g.sources[i].y;
      sources[3 * i + 2] = g.sources[i].z;
      angles[i] = g.angles[i];
    }
  });
}

int ref_cone_from_matrices(const or_volume* vol, const or_det2* det, uint64_t n, double range,
                           double sid, double sdd, const double* mats_in, double* mats,
                           double* sources, double* invs, double* angles) {
  return guard([&] {
    std::vector<Mat34> m(n);
    for (std::size_t i = 0; i < n; ++i)
      for (int k = 0; k < 12; ++k) m[i].m[std::size_t(k)] = mats_in[12 * i + std::size_t(k)];
    auto g = make_cone_from_matrices(to_spec(*vol), to_det(*det), range, sid, sdd, m);
    for (std::size_t i = 0; i < n; ++i) {
      std::memcpy(mats + 12 * i, g.matrices[i].m.data(), 12 * sizeof(double));
      std::memcpy(invs + 9 * i, g.inv_blocks[i].m.data(), 9 * sizeof(double));
      sources[3 * i] = g.sources[i].x;
      sources[3 * i + 1] = g.sources[i].y;
      sources[3 * i + 2] = g.sources[i].z;
      angles[i] = g.angles[i];
    }
  });
}

int ref_planar_rays(const or_volume* vol, const or_det1* det, uint64_t n, double range, double sid,
                    double sdd, double* rays, double* angles) {
  return guard([&] {
    std::vector<Vec2> r;
    std::vector<double> a;
    if (sdd > 0.0) {
      auto g = make_fan(to_spec(*vol), to_det(*det), std::size_t(n), range, sid, sdd);
      r = g.rays;
      a = g.angles;
    } else {
      auto g = make_parallel(to_spec(*vol), to_det(*det), std::size_t(n), range);
      r = g.rays;
      a = g.angles;
    }
    for (std::size_t i = 0; i < n; ++i) {
      rays[2 * i] = r[i].x;
      rays[2 * i + 1] = r[i].y;
      angles[i] = a[i];
    }
  });
}

#define REF_OPS(SUF, T)                                                                       \
  int ref_planar_forward_##SUF(const or_planar* g, const T* img, T* sino) {                   \
    return guard([&] {                                                                        \
      auto im = make_image<T>(to_spec(g->vol), img);                                          \
      Sinogram<T> s = g->sdd > 0.0 ? forward_project(im, to_fan(*g))                          \
                                   : forward_project(im, to_parallel(*g));                    \
      std::memcpy(sino, s.data.data(), sizeof(T) * s.data.size());                            \
    });                                                                                       \
  }                                                                                           \
  int ref_planar_backproject_##SUF(const or_planar* g, const T* sino, T* img) {               \
    return guard([&] {                                                                        \
      auto s = Sinogram<T>::planar(std::size_t(g->n_proj), to_det(g->det));                  \
      std::memcpy(s.data.data(), sino, sizeof(T) * s.data.size());                            \
      Image<T> im = g->sdd > 0.0 ? back_project(s, to_fan(*g)) : back_project(s, to_parallel(*g)); \
      std::memcpy(img, im.data.data(), sizeof(T) * im.data.size());                           \
    });                                                                                       \
  }                                                                                           \
  int ref_cone_forward_##SUF(const or_cone* g, int circular, const T* vol, T* sino) {         \
    return guard([&] {                                                                        \
      auto im = make_image<T>(to_spec(g->vol), vol);                                          \
      auto s = forward_project(im, to_cone(*g, circular != 0));                               \
      std::memcpy(sino, s.data.data(), sizeof(T) * s.data.size());                            \
    });                                                                                       \
  }                                                                                           \
  int ref_cone_backproject_##SUF(const or_cone* g, int circular, const T* sino, T* vol) {     \
    return guard([&] {                                                                        \
      auto s = Sinogram<T>::cone_beam(std::size_t(g->n_proj), to_det(g->det));               \
      std::memcpy(s.data.data(), sino, sizeof(T) * s.data.size());                            \
      auto im = back_project(s, to_cone(*g, circular != 0));                                  \
      std::memcpy(vol, im.data.data(), sizeof(T) * im.data.size());                           \
    });                                                                                       \
  }                                                                                           \
  int ref_fdk_reconstruct_##SUF(const or_cone* g, int circular, const T* sino, T* vol,        \
                                int use_parker) {                                             \
    return guard([&] {                                                                        \
      auto s = Sinogram<T>::cone_beam(std::size_t(g->n_proj), to_det(g->det));               \
      std::memcpy(s.data.data(), sino, sizeof(T) * s.data.size());                            \
      auto im = fdk_reconstruct(s, to_cone(*g, circular != 0), use_parker != 0);              \
      std::memcpy(vol, im.data.data(), sizeof(T) * im.data.size());                           \
    });                                                                                       \
  }                                                                                           \
  int ref_fbp_reconstruct_##SUF(const or_planar* g, const T* sino, T* img, int ramlak) {      \
    return guard([&] {                                                                        \
      auto s = Sinogram<T>::planar(std::size_t(g->n_proj), to_det(g->det));                  \
      std::memcpy(s.data.data(), sino, sizeof(T) * s.data.size());                            \
      auto im = fbp_reconstruct(s, to_parallel(*g), ramlak ? FilterKind::ramlak : FilterKind::ramp); \
      std::memcpy(img, im.data.data(), sizeof(T) * im.data.size());                           \
    });                                                                                       \
  }                                                                                           \
  /* apply_filter on n_rows planar rows of n bins (spacing ds) with explicit weights */      \
  int ref_apply_filter_##SUF(T* data, uint64_t n_rows, uint64_t n, double ds,                 \
                             const double* weights, uint64_t padded_n, uint64_t n_weights) {  \
    return guard([&] {                                                                        \
      auto s = Sinogram<T>::planar(std::size_t(n_rows), Detector1D::centered(std::size_t(n), ds)); \
      std::memcpy(s.data.data(), data, sizeof(T) * s.data.size());                            \
      Filter1D f{std::size_t(n), std::size_t(padded_n), ds,                                   \
                 std::vector<double>(weights, weights + n_weights)};                          \
      auto o = apply_filter(s, f);                                                            \
      std::memcpy(data, o.data.data(), sizeof(T) * o.data.size());                            \
    });                                                                                       \
  }                                                                                           \
  int ref_shepp_logan_3d_##SUF(const or_volume* vol, T* out) {                               \
    return guard([&] {                                                                        \
      auto im = shepp_logan_3d<T>(to_spec(*vol));                                             \
      std::memcpy(out, im.data.data(), sizeof(T) * im.data.size());                           \
    });                                                                                       \
  }                                                                                           \
  int ref_shepp_logan_2d_##SUF(const or_volume* vol, T* out) {                               \
    return guard([&] {                                                                        \
      auto im = shepp_logan_2d<T>(to_spec(*vol));                                             \
      std::memcpy(out, im.data.data(), sizeof(T) * im.data.size());                           \
    });                                                                                       \
  }

REF_OPS(f32, float)
REF_OPS(f64, double)

int ref_ramlak_weights(uint64_t padded_n, double spacing, double* out) {
  return guard([&] {
    auto w = ramlak_weights(std::size_t(padded_n), spacing);
    std::memcpy(out, w.data(), sizeof(double) * w.size());
  });
}

int ref_ramp_weights(uint64_t padded_n, double spacing, double* out) {
  return guard([&] {
    auto w = ramp_weights(std::size_t(padded_n), spacing);
    std::memcpy(out, w.data(), sizeof(double) * w.size());
  });
}

int ref_cosine_weights_cone(const or_cone* g, double* out) {
  return guard([&] {
    auto m = cosine_weights(to_cone(*g, true));
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
  });
}

// compact [view][u] copy of the reference's full [view][v][u] Parker map
int ref_parker_weights_cone(const or_cone* g, double* out) {
  return guard([&] {
    auto geo = to_cone(*g, true);
    auto m = parker_weights(geo);
    const std::size_t nu = g->det.n_u, nv = g->det.n_v;
    for (std::size_t i = 0; i < g->n_proj; ++i)
      std::memcpy(out + i * nu, m.data.data() + i * nv * nu, sizeof(double) * nu);
  });
}

int ref_parker_weights_fan(const or_planar* g, double* out) {
  return guard([&] {
    auto m = parker_weights(to_fan(*g));
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
  });
}

int ref_cosine_weights_fan(const or_planar* g, double* out) {
  return guard([&] {
    auto m = cosine_weights(to_fan(*g));
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
  });
}

}  // extern "C"
