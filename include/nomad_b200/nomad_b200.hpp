// nomad_b200.hpp — header-only C++ shim that re-exposes the reference
// library's hot-path signatures (/root/reference/proj/include/nomad) on top of
// the C-ABI in nomad_b200.h. A reference caller switches by including this
// header next to "nomad/nomad.hpp" and calling nomad::b200::X instead of
// nomad::X. Types are the reference's own
// (VectorDataset, ClusterAssignment, KnnGraph, LayoutMatrix, TrainConfig,
// FitReport); errors come back as nomad::Error with the same ErrorKind and
// message text.
//
//   reference                                         shim
//   lsh_init            kmeans.hpp:167-168            nomad::b200::lsh_init
//   kmeans_em           kmeans.hpp:257-261            nomad::b200::kmeans_em
//   default_kmeans_tol  kmeans.hpp:157                nomad::b200::default_kmeans_tol
//   build_knn           knn.hpp:65-66                 nomad::b200::build_knn
//   pca_init            pca.hpp:79                    nomad::b200::pca_init
//   fit                 optimizer.hpp:327-328         nomad::b200::fit
//   neighborhood_preservation metrics.hpp:113         nomad::b200::neighborhood_preservation
//   random_triplet_accuracy   metrics.hpp:205         nomad::b200::random_triplet_accuracy
//   load_vectors_raw    dataset.hpp:122-125           nomad::b200::load_vectors_raw
//   save_layout         dataset.hpp:223-226           nomad::b200::save_layout
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "nomad/nomad.hpp"
#include "nomad_b200.h"

namespace nomad::b200 {

/// Engine-only knobs (not part of the reference's TrainConfig).
struct EngineOptions {
  int device = 0;
  int sgd_mode = NOMAD_B200_SGD_REPLAY;  // bit-exact replay by default
  int knn_mode = NOMAD_B200_KNN_EXACT;
  unsigned hogwild_cap = 0;
  bool hogwild_double_float = false;
};

inline EngineOptions& options() {
  static thread_local EngineOptions o;
  return o;
}

namespace detail {

inline void check(int32_t rc) {
  if (rc != NOMAD_B200_OK)
    throw nomad::Error(static_cast<nomad::ErrorKind>(rc - 1), nomad_b200_last_error());
}

/// One context per (thread, device), created on first use.
inline nomad_b200_ctx* ctx() {
  struct Holder {
    nomad_b200_ctx* c = nullptr;
    int dev = -1;
    ~Holder() {
      if (c) nomad_b200_destroy(c);
    }
  };
  static thread_local Holder h;
  if (!h.c || h.dev != options().device) {
    if (h.c) nomad_b200_destroy(h.c);
    h.c = nullptr;
    check(nomad_b200_create(options().device, &h.c));
    h.dev = options().device;
  }
  return h.c;
}

inline nomad_b200_dataset_view view(const VectorDataset& d) {
  return nomad_b200_dataset_view{d.rows, d.dims, d.data.data(), NOMAD_B200_HOST, NOMAD_B200_F32};
}

inline nomad_b200_clusters cview(ClusterAssignment& ca, std::size_t rows) {
  return nomad_b200_clusters{rows,
                             ca.n_clusters,
                             ca.dims,
                             ca.assignment.data(),
                             ca.centroids.data(),
                             ca.sizes.data(),
                             NOMAD_B200_HOST};
}

inline nomad_b200_train_config cfg(const TrainConfig& c) {
  nomad_b200_train_config o;
  nomad_b200_default_config(&o);
  o.epochs = c.epochs;
  o.k = c.k;
  o.negatives = c.negatives;
  o.local_draws = c.local_draws;
  o.batch_size = c.batch_size;
  o.workers = c.workers;
  o.n_clusters = c.n_clusters;
  o.seed = c.seed;
  o.lr0 = c.lr0;
  o.kmeans_max_iters = c.kmeans_max_iters;
  o.kmeans_tol = c.kmeans_tol;
  o.approx_all_but_own = c.approx == ApproxMode::AllButOwnCluster ? 1 : 0;
  o.head_only = c.head_only ? 1 : 0;
  o.checkpoint_every = c.checkpoint_every;
  o.checkpoint_prefix = c.checkpoint_prefix.c_str();  // valid while c lives
  o.verbose = c.verbose ? 1 : 0;
  o.sgd_mode = options().sgd_mode;
  o.knn_mode = options().knn_mode;
  o.hogwild_cap = options().hogwild_cap;
  o.hogwild_double_float = options().hogwild_double_float ? 1 : 0;
  return o;
}

}  // namespace detail

/// kmeans.hpp:157-161
inline double default_kmeans_tol(const VectorDataset& data) {
  double t = 0.0;
  const auto v = detail::view(data);
  detail::check(nomad_b200_default_kmeans_tol(detail::ctx(), &v, &t));
  return t;
}

/// kmeans.hpp:167-250
inline ClusterAssignment lsh_init(const VectorDataset& data, std::size_t n_clusters,
                                  std::uint64_t seed) {
  ClusterAssignment ca;
  ca.n_clusters = n_clusters;
  ca.dims = data.dims;
  ca.assignment.assign(data.rows, 0);
  ca.centroids.assign(n_clusters * data.dims, 0.0);
  ca.sizes.assign(n_clusters, 0);
  const auto v = detail::view(data);
  auto cv = detail::cview(ca, data.rows);
  detail::check(nomad_b200_lsh_init(detail::ctx(), &v, n_clusters, seed, &cv));
  return ca;
}

/// kmeans.hpp:257-296 (init taken by value, as the reference)
inline ClusterAssignment kmeans_em(const VectorDataset& data, ClusterAssignment init,
                                   std::size_t max_iters = 100, double tol = 0.0,
                                   std::vector<double>* qe_trace = nullptr) {
  if (init.assignment.size() != data.rows || init.dims != data.dims)
    fail(ErrorKind::Parameter, "init assignment does not match dataset");
  const auto v = detail::view(data);
  auto cv = detail::cview(init, data.rows);
  std::vector<double> trace(max_iters > 0 ? max_iters : 1);
  std::uint64_t iters = 0;
  detail::check(nomad_b200_kmeans_em(detail::ctx(), &v, &cv, max_iters, tol,
                                     qe_trace ? trace.data() : nullptr, &iters));
  if (qe_trace) qe_trace->assign(trace.begin(), trace.begin() + iters);
  return init;
}

/// knn.hpp:65-109
inline KnnGraph build_knn(const VectorDataset& data, const ClusterAssignment& clusters,
                          std::size_t k) {
  if (k < 1) fail(ErrorKind::Parameter, "k must be >= 1");
  KnnGraph g;
  g.rows = data.rows;
  g.k = k;
  g.offsets.assign(data.rows + 1, 0);
  g.neighbors.assign(data.rows * k, 0);
  g.distances.assign(data.rows * k, 0.0);
  const auto v = detail::view(data);
  ClusterAssignment c = clusters;
  auto cv = detail::cview(c, data.rows);
  nomad_b200_graph gv{data.rows, k, g.offsets.data(), g.neighbors.data(), g.distances.data(),
                      NOMAD_B200_HOST};
  detail::check(nomad_b200_build_knn(detail::ctx(), &v, &cv, k, options().knn_mode, &gv));
  g.neighbors.resize(g.offsets[data.rows]);
  g.distances.resize(g.offsets[data.rows]);
  return g;
}

/// pca.hpp:79-218 (GPU; bit-identical)
inline LayoutMatrix pca_init(const VectorDataset& data, std::uint64_t seed = 0) {
  LayoutMatrix l = LayoutMatrix::zeros(data.rows);
  const auto v = detail::view(data);
  detail::check(nomad_b200_pca_init(detail::ctx(), &v, seed, l.positions.data(),
                                    NOMAD_B200_HOST));
  return l;
}

/// optimizer.hpp:327-482. The report's affinity / plan / final means are
/// rebuilt on the host from the engine's clusters and graph with the
/// reference's own build_affinity / shard_clusters / gather_means.
inline LayoutMatrix fit(const VectorDataset& data, const TrainConfig& config,
                        FitReport* report = nullptr) {
  config.validate();
  const std::size_t n = data.rows;
  const std::size_t C = config.resolve_clusters(n);
  const LayoutMatrix pca = nomad::b200::pca_init(data, config.seed);
  LayoutMatrix out = LayoutMatrix::zeros(n);
  ClusterAssignment ca;
  ca.n_clusters = C;
  ca.dims = data.dims;
  ca.assignment.assign(n, 0);
  ca.centroids.assign(C * data.dims, 0.0);
  ca.sizes.assign(C, 0);
  KnnGraph g;
  g.rows = n;
  g.k = config.k;
  g.offsets.assign(n + 1, 0);
  g.neighbors.assign(n * config.k, 0);
  g.distances.assign(n * config.k, 0.0);
  std::vector<double> losses(config.epochs > 0 ? config.epochs : 1);
  const auto v = detail::view(data);
  auto cv = detail::cview(ca, n);
  nomad_b200_graph gv{n, config.k, g.offsets.data(), g.neighbors.data(), g.distances.data(),
                      NOMAD_B200_HOST};
  auto c = detail::cfg(config);
  // checkpoint rows carry the dataset's ids / labels, as save_layout does
  std::vector<const char*> idp, lbp;
  for (const auto& s : data.ids) idp.push_back(s.c_str());
  for (const auto& s : data.labels) lbp.push_back(s.c_str());
  c.checkpoint_ids = idp.size() == n ? idp.data() : nullptr;
  c.checkpoint_labels = lbp.size() == n ? lbp.data() : nullptr;
  detail::check(nomad_b200_fit(detail::ctx(), &v, &c, pca.positions.data(),
                               out.positions.data(), &cv, &gv, losses.data()));
  out.epoch = config.epochs;
  if (report) {
    g.neighbors.resize(g.offsets[n]);
    g.distances.resize(g.offsets[n]);
    report->clusters = ca;
    report->graph = g;
    report->affinity = nomad::build_affinity(g);
    report->plan = nomad::shard_clusters(ca, config.workers);
    report->pca = pca;
    report->final_means = nomad::gather_means(out, ca, config.epochs);
    report->comm.epochs.assign(config.epochs, {});
    for (auto& msgs : report->comm.epochs)
      for (std::size_t w = 0; w < config.workers; ++w) {
        MeansMessage m;
        m.worker = static_cast<std::uint32_t>(w);
        m.clusters = static_cast<std::uint32_t>(report->plan.worker_clusters[w].size());
        m.payload_doubles = 2ull * m.clusters;
        m.payload_counts = m.clusters;
        msgs.push_back(m);
      }
    report->epoch_mean_loss.assign(losses.begin(), losses.begin() + config.epochs);
  }
  return out;
}

/// metrics.hpp:113-168 on the GPU (bit-identical value and std_error; k <= 56)
inline MetricReport neighborhood_preservation(const VectorDataset& high, const LayoutMatrix& low,
                                              std::size_t k, std::size_t sample = 0,
                                              std::uint64_t seed = 0) {
  if (low.rows != high.rows) fail(ErrorKind::Parameter, "vector and layout row counts differ");
  MetricReport r;
  r.metric = "np";
  r.param = k;
  r.sample = (sample == 0 || sample >= high.rows) ? 0 : sample;
  r.seed = seed;
  const auto v = detail::view(high);
  detail::check(nomad_b200_neighborhood_preservation(detail::ctx(), &v, low.positions.data(),
                                                     NOMAD_B200_HOST, k, sample, seed, &r.value,
                                                     &r.std_error));
  return r;
}

/// metrics.hpp:205-243 on the GPU (bit-identical)
inline MetricReport random_triplet_accuracy(const VectorDataset& high, const LayoutMatrix& low,
                                            std::size_t n_triplets, std::uint64_t seed = 0) {
  if (low.rows != high.rows) fail(ErrorKind::Parameter, "vector and layout row counts differ");
  MetricReport r;
  r.metric = "triplet";
  r.param = n_triplets;
  r.seed = seed;
  const auto v = detail::view(high);
  detail::check(nomad_b200_random_triplet_accuracy(detail::ctx(), &v, low.positions.data(),
                                                   NOMAD_B200_HOST, n_triplets, seed, &r.value,
                                                   &r.std_error));
  return r;
}

/// dataset.hpp:122-173 (host result; default ids)
inline VectorDataset load_vectors_raw(const std::string& path, std::optional<std::size_t> rows,
                                      std::optional<std::size_t> dims) {
  std::uint64_t n = 0, d = 0;
  detail::check(nomad_b200_load_vectors_raw(nullptr, path.c_str(), rows.value_or(0),
                                            dims.value_or(0), nullptr, NOMAD_B200_HOST, &n, &d));
  VectorDataset ds;
  ds.rows = n;
  ds.dims = d;
  ds.data.resize(n * d);
  detail::check(nomad_b200_load_vectors_raw(nullptr, path.c_str(), n, d, ds.data.data(),
                                            NOMAD_B200_HOST, nullptr, nullptr));
  ds.ids.resize(n);
  for (std::size_t i = 0; i < n; ++i) ds.ids[i] = std::to_string(i);
  return ds;
}

/// dataset.hpp:223-250 (byte-identical CSV, formatted on all host cores)
inline void save_layout(const LayoutMatrix& layout, const std::vector<std::string>& ids,
                        const std::vector<std::string>& labels, const std::string& path) {
  if (ids.size() != layout.rows)
    fail(ErrorKind::Parameter, "ids length " + std::to_string(ids.size()) + " != layout rows " +
                                   std::to_string(layout.rows));
  if (!labels.empty() && labels.size() != layout.rows)
    fail(ErrorKind::Parameter, "labels length != layout rows");
  std::vector<const char*> ip, lp;
  for (const auto& x : ids) ip.push_back(x.c_str());
  for (const auto& x : labels) lp.push_back(x.c_str());
  detail::check(nomad_b200_save_layout_csv(path.c_str(), layout.positions.data(), layout.rows,
                                           ip.data(), labels.empty() ? nullptr : lp.data()));
}

}  // namespace nomad::b200
