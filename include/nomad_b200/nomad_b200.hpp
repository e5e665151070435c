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
  /// fit() over several GPUs from this one call (the reference runs its W
  /// workers from one fit() call, optimizer.hpp:399-408): empty = {device}.
  /// Distinct devices: NCCL; one device repeated: loopback ranks on it.
  std::vector<int> devices;
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

/// The group over options().devices (created on first use, per thread).
inline nomad_b200_group* group() {
  struct Holder {
    nomad_b200_group* g = nullptr;
    std::vector<int> devs;
    ~Holder() {
      if (g) nomad_b200_group_destroy(g);
    }
  };
  static thread_local Holder h;
  const auto& want = options().devices;
  if (!h.g || h.devs != want) {
    if (h.g) nomad_b200_group_destroy(h.g);
    h.g = nullptr;
    std::vector<int32_t> d(want.begin(), want.end());
    check(nomad_b200_group_create(d.data(), (int32_t)d.size(), &h.g));
    h.devs = want;
  }
  return h.g;
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

/// optimizer.hpp:327-482. Every FitReport field comes from the engine: the
/// index, the PCA the epochs started from (bit-identical in replay mode, the
/// precomputed-covariance form in throughput mode), the affinity weights and
/// eligible heads, the shard plan, the last all-gathered means and CommLog.
inline LayoutMatrix fit(const VectorDataset& data, const TrainConfig& config,
                        FitReport* report = nullptr) {
  config.validate();
  const std::size_t n = data.rows;
  const std::size_t C = config.resolve_clusters(n);
  LayoutMatrix out = LayoutMatrix::zeros(n);
  ClusterAssignment ca;
  KnnGraph g;
  LayoutMatrix pca;
  std::vector<double> losses, means, weights;
  std::vector<std::uint32_t> c2w, elig;
  nomad_b200_clusters cv{};
  nomad_b200_graph gv{};
  nomad_b200_fit_report rep{};
  if (report) {  // the full outputs only when asked for (12 n k bytes of graph)
    ca.n_clusters = C;
    ca.dims = data.dims;
    ca.assignment.assign(n, 0);
    ca.centroids.assign(C * data.dims, 0.0);
    ca.sizes.assign(C, 0);
    g.rows = n;
    g.k = config.k;
    g.offsets.assign(n + 1, 0);
    g.neighbors.assign(n * config.k, 0);
    g.distances.assign(n * config.k, 0.0);
    pca = LayoutMatrix::zeros(n);
    losses.assign(config.epochs > 0 ? config.epochs : 1, 0.0);
    means.assign(2 * C, 0.0);
    weights.assign(n * config.k, 0.0);
    c2w.assign(C, 0);
    elig.assign(n, 0);
    cv = detail::cview(ca, n);
    gv = nomad_b200_graph{n, config.k, g.offsets.data(), g.neighbors.data(), g.distances.data(),
                          NOMAD_B200_HOST};
    rep.clusters = &cv;
    rep.graph = &gv;
    rep.epoch_mean_loss = losses.data();
    rep.pca = pca.positions.data();
    rep.final_means = means.data();
    rep.cluster_to_worker = c2w.data();
    rep.affinity_weights = weights.data();
    rep.eligible_heads = elig.data();
  }
  const auto v = detail::view(data);
  auto c = detail::cfg(config);
  // checkpoint rows carry the dataset's ids / labels, as save_layout does
  std::vector<const char*> idp, lbp;
  for (const auto& s : data.ids) idp.push_back(s.c_str());
  for (const auto& s : data.labels) lbp.push_back(s.c_str());
  c.checkpoint_ids = idp.size() == n ? idp.data() : nullptr;
  c.checkpoint_labels = lbp.size() == n ? lbp.data() : nullptr;
  const bool multi = options().devices.size() > 1;
  detail::check(nomad_b200_fit_ex(multi ? nullptr : detail::ctx(), multi ? detail::group() : nullptr,
                                  &v, &c, nullptr, out.positions.data(), report ? &rep : nullptr));
  out.epoch = config.epochs;
  if (report) {
    g.neighbors.resize(g.offsets[n]);
    g.distances.resize(g.offsets[n]);
    weights.resize(g.offsets[n]);
    elig.resize(rep.n_eligible);
    report->clusters = ca;
    report->affinity.rows = n;
    report->affinity.offsets = g.offsets;
    report->affinity.neighbors = g.neighbors;
    report->affinity.weights = std::move(weights);
    report->affinity.eligible_heads = std::move(elig);
    report->graph = std::move(g);
    // ShardPlan (optimizer.hpp:94-144) from the engine's cluster -> worker map
    ShardPlan& P = report->plan;
    P.workers = config.workers;
    P.cluster_to_worker = c2w;
    P.worker_clusters.assign(config.workers, {});
    P.worker_points.assign(config.workers, {});
    P.worker_point_counts.assign(config.workers, 0);
    for (std::size_t r = 0; r < C; ++r) P.worker_clusters[c2w[r]].push_back((std::uint32_t)r);
    for (std::size_t i = 0; i < n; ++i) {
      const std::uint32_t w = c2w[ca.assignment[i]];
      P.worker_points[w].push_back((std::uint32_t)i);
      ++P.worker_point_counts[w];
    }
    report->pca = std::move(pca);
    report->final_means.means = std::move(means);
    report->final_means.counts = ca.sizes;
    report->final_means.epoch_stamp = config.epochs;
    report->comm.epochs.assign(config.epochs, {});
    for (auto& msgs : report->comm.epochs)
      for (std::size_t w = 0; w < config.workers; ++w) {
        MeansMessage m;
        m.worker = static_cast<std::uint32_t>(w);
        m.clusters = static_cast<std::uint32_t>(P.worker_clusters[w].size());
        m.payload_doubles = 2ull * m.clusters;
        m.payload_counts = m.clusters;
        msgs.push_back(m);
      }
    report->epoch_mean_loss.assign(losses.begin(), losses.begin() + config.epochs);
  }
  return out;
}

/// metrics.hpp:113-168 on the GPU (bit-identical value and std_error; k <= 1024)
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
