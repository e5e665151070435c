// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product.
//
// A thin extern "C" driver around the UNMODIFIED reference library
// (/root/reference/proj/include/nomad/*.hpp, header-only C++20). It is built
// by oracle/Makefile into oracle/_ref/libnomad_ref.so (git-ignored) with the
// pinned flags -O2 -std=c++20 -ffp-contract=off (FMA
// contraction changes reference bits). Nothing here re-implements reference
// math: every function forwards to the reference's own entry point, so the
// outputs are the reference's outputs. Uses:
//   * pin the C restatement (oracle/nomad_oracle.c) and generate golden
//     fixtures (tests/golden/, tests/make_golden.py);
//   * bench.py's cpu_baseline / --impl reference arm: the reference's own
//     detail::run_worker_epoch on W std::threads, as fit() runs it
//     (optimizer.hpp:399-408).
//
// Error convention (mirrors the product C-ABI): 0 = ok, else 1 + ErrorKind
// (error.hpp:25-36); message via ref_last_error().

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "nomad/nomad.hpp"

namespace {

thread_local std::string g_err;

int fail_code(const nomad::Error& e) {
  g_err = e.what();
  return 1 + static_cast<int>(e.kind());
}

nomad::VectorDataset make_ds(const float* data, uint64_t n, uint64_t d) {
  nomad::VectorDataset ds;
  ds.rows = n;
  ds.dims = d;
  ds.data.assign(data, data + n * d);
  return ds;
}

nomad::ClusterAssignment make_ca(uint64_t n, uint64_t d, uint64_t C,
                                 const uint32_t* assign, const double* centroids,
                                 const uint32_t* sizes) {
  nomad::ClusterAssignment ca;
  ca.n_clusters = C;
  ca.dims = d;
  ca.assignment.assign(assign, assign + n);
  if (centroids) ca.centroids.assign(centroids, centroids + C * d);
  else ca.centroids.assign(C * d, 0.0);
  if (sizes) {
    ca.sizes.assign(sizes, sizes + C);
  } else {
    ca.sizes.assign(C, 0);
    for (uint64_t i = 0; i < n; ++i) ++ca.sizes[assign[i]];
  }
  return ca;
}

void export_ca(const nomad::ClusterAssignment& ca, uint32_t* assign,
               double* centroids, uint32_t* sizes) {
  if (assign) std::memcpy(assign, ca.assignment.data(), ca.assignment.size() * 4);
  if (centroids)
    std::memcpy(centroids, ca.centroids.data(), ca.centroids.size() * 8);
  if (sizes) std::memcpy(sizes, ca.sizes.data(), ca.sizes.size() * 4);
}

}  // namespace

extern "C" {

struct ref_train_config {
  uint64_t epochs, k, negatives, local_draws, batch_size, workers, n_clusters;
  uint64_t seed;
  double lr0;
  uint64_t kmeans_max_iters;
  double kmeans_tol;
  int32_t approx_all_but_own;  // ApproxMode::AllButOwnCluster
  int32_t head_only;
};

const char* ref_last_error(void) { return g_err.c_str(); }

// rng.hpp:25-84 known answers and draw streams.
uint64_t ref_stream_seed(uint64_t base, uint64_t stream) {
  return nomad::stream_seed(base, stream);
}
void ref_rng_u64(uint64_t seed, uint64_t count, uint64_t* out) {
  nomad::Rng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}
void ref_rng_gaussian(uint64_t seed, uint64_t count, double* out) {
  nomad::Rng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.gaussian();
}
void ref_rng_uniform_index(uint64_t seed, uint64_t bound, uint64_t count,
                           uint64_t* out) {
  nomad::Rng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.uniform_index(bound);
}

int ref_inverse_rank_weights(uint64_t k, double* out) {
  try {
    auto w = nomad::inverse_rank_weights(k);
    std::memcpy(out, w.data(), k * 8);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

double ref_lr_schedule(uint64_t epoch, uint64_t total, double lr0) {
  return nomad::lr_schedule(epoch, total, lr0);
}

// Per-row checkers for configurations too large for the whole reference
// build (1M-10M rows): the reference's own distance functions and selection
// rule applied to a row sample.
//
// knn.hpp:51-58, :88-106 — for each query (an index into `members`, the rows
// of one cluster in ascending point id), the min(k, m - 1) smallest
// (detail::sq_dist_ff, id) pairs over the other members, by std::partial_sort
// on std::pair<double, uint32_t> exactly as build_knn selects them.
int ref_knn_rows(const float* members, const uint32_t* ids, uint64_t m, uint64_t d,
                 const uint64_t* queries, uint64_t nq, uint64_t k, uint32_t* out_ids,
                 double* out_dist, int32_t threads) {
  const uint64_t want = std::min<uint64_t>(k, m ? m - 1 : 0);
  auto one = [&](uint64_t q) {
    const uint64_t qi = queries[q];
    std::vector<std::pair<double, std::uint32_t>> cand;
    cand.reserve(m);
    for (uint64_t j = 0; j < m; ++j) {
      if (j == qi) continue;
      cand.emplace_back(nomad::detail::sq_dist_ff(members + qi * d, members + j * d, d), ids[j]);
    }
    std::partial_sort(cand.begin(), cand.begin() + want, cand.end());
    for (uint64_t t = 0; t < want; ++t) {
      out_ids[q * k + t] = cand[t].second;
      out_dist[q * k + t] = cand[t].first;
    }
  };
  const uint64_t nt = std::max<int32_t>(1, threads);
  std::vector<std::thread> pool;
  for (uint64_t t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (uint64_t q = t; q < nq; q += nt) one(q);
    });
  for (auto& x : pool) x.join();
  return (int)want;
}

// kmeans.hpp:47-68 detail::nearest_centroid for a set of rows.
void ref_nearest_centroid_rows(const float* rows, uint64_t nr, uint64_t d,
                               const double* centroids, uint64_t C, uint32_t* out,
                               int32_t threads) {
  nomad::ClusterAssignment ca;
  ca.n_clusters = C;
  ca.dims = d;
  ca.centroids.assign(centroids, centroids + C * d);
  const uint64_t nt = std::max<int32_t>(1, threads);
  std::vector<std::thread> pool;
  for (uint64_t t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (uint64_t i = t; i < nr; i += nt) out[i] = nomad::detail::nearest_centroid(ca, rows + i * d);
    });
  for (auto& x : pool) x.join();
}

// kmeans.hpp:75-88 detail::recompute_centroid of one cluster, given only its
// member rows in ascending point id (the other rows are skipped by the
// reference's pass and do not change the sums).
void ref_cluster_centroid(const float* members, uint64_t m, uint64_t d, double* out) {
  nomad::VectorDataset ds = make_ds(members, m, d);
  nomad::ClusterAssignment ca;
  ca.n_clusters = 1;
  ca.dims = d;
  ca.assignment.assign(m, 0);
  ca.centroids.assign(d, 0.0);
  nomad::detail::recompute_centroid(ds, ca, 0);
  std::memcpy(out, ca.centroids.data(), d * 8);
}

// kmeans.hpp:157-161
double ref_default_kmeans_tol(const float* data, uint64_t n, uint64_t d) {
  return nomad::default_kmeans_tol(make_ds(data, n, d));
}

// kmeans.hpp:167-250
int ref_lsh_init(const float* data, uint64_t n, uint64_t d, uint64_t C,
                 uint64_t seed, uint32_t* assign, double* centroids,
                 uint32_t* sizes) {
  try {
    auto ca = nomad::lsh_init(make_ds(data, n, d), C, seed);
    export_ca(ca, assign, centroids, sizes);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// kmeans.hpp:257-296; qe_trace (nullable) must hold max_iters doubles.
int ref_kmeans_em(const float* data, uint64_t n, uint64_t d, uint64_t C,
                  uint32_t* assign, double* centroids, uint32_t* sizes,
                  uint64_t max_iters, double tol, double* qe_trace,
                  uint64_t* n_trace) {
  try {
    auto ds = make_ds(data, n, d);
    auto init = make_ca(n, d, C, assign, centroids, sizes);
    std::vector<double> trace;
    auto ca = nomad::kmeans_em(ds, std::move(init), max_iters, tol,
                               qe_trace ? &trace : nullptr);
    export_ca(ca, assign, centroids, sizes);
    if (qe_trace) std::memcpy(qe_trace, trace.data(), trace.size() * 8);
    if (n_trace) *n_trace = trace.size();
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// knn.hpp:65-109. offsets: n+1; neighbors/distances: offsets[n] entries
// (callers size them n*k).
int ref_build_knn(const float* data, uint64_t n, uint64_t d, uint64_t C,
                  const uint32_t* assign, uint64_t k, uint32_t* offsets,
                  uint32_t* neighbors, double* distances) {
  try {
    auto ds = make_ds(data, n, d);
    auto ca = make_ca(n, d, C, assign, nullptr, nullptr);
    auto g = nomad::build_knn(ds, ca, k);
    std::memcpy(offsets, g.offsets.data(), (n + 1) * 4);
    std::memcpy(neighbors, g.neighbors.data(), g.neighbors.size() * 4);
    std::memcpy(distances, g.distances.data(), g.distances.size() * 8);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// pca.hpp:79-218
int ref_pca_init(const float* data, uint64_t n, uint64_t d, uint64_t seed,
                 double* layout) {
  try {
    auto l = nomad::pca_init(make_ds(data, n, d), seed);
    std::memcpy(layout, l.positions.data(), n * 2 * 8);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// optimizer.hpp:149-176
int ref_gather_means(const double* layout, uint64_t n, uint64_t C,
                     const uint32_t* assign, double* means) {
  try {
    nomad::LayoutMatrix l;
    l.rows = n;
    l.positions.assign(layout, layout + 2 * n);
    auto ca = make_ca(n, 1, C, assign, nullptr, nullptr);
    auto m = nomad::gather_means(l, ca, 0);
    std::memcpy(means, m.means.data(), C * 2 * 8);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// optimizer.hpp:106-144. worker_points_out: n entries, worker-major, each
// worker's points ascending; worker_offsets: W+1.
int ref_shard_clusters(uint64_t n, uint64_t C, const uint32_t* assign,
                       uint64_t W, uint32_t* cluster_to_worker,
                       uint32_t* worker_points_out, uint64_t* worker_offsets) {
  try {
    auto ca = make_ca(n, 1, C, assign, nullptr, nullptr);
    auto plan = nomad::shard_clusters(ca, W);
    std::memcpy(cluster_to_worker, plan.cluster_to_worker.data(), C * 4);
    uint64_t off = 0;
    for (uint64_t w = 0; w < W; ++w) {
      worker_offsets[w] = off;
      for (uint32_t i : plan.worker_points[w]) worker_points_out[off++] = i;
    }
    worker_offsets[W] = off;
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// objective.hpp:178-237 for one head (gradient unit tests).
// grads: 2*(1 + nn + s) doubles: head, neighbors..., negatives...
int ref_nomad_gradient(const double* layout, uint64_t n, uint32_t head,
                       const uint32_t* nbrs, const double* weights, uint64_t nn,
                       const uint32_t* negs, uint64_t s, const uint32_t* remote,
                       const double* remote_probs, uint64_t nr,
                       const double* means, uint64_t C, double local_mass,
                       uint64_t m_total, double* loss, double* grads) {
  try {
    nomad::LayoutMatrix l;
    l.rows = n;
    l.positions.assign(layout, layout + 2 * n);
    nomad::ClusterMeans cm;
    cm.means.assign(means, means + 2 * C);
    cm.counts.assign(C, 1);
    nomad::LossBatchSpec spec;
    spec.head = head;
    spec.neighbors = {nbrs, nn};
    spec.weights = {weights, nn};
    spec.negatives = {negs, s};
    spec.remote_cells = {remote, nr};
    spec.remote_probs = {remote_probs, nr};
    spec.local_mass = local_mass;
    spec.m_total = m_total;
    auto g = nomad::nomad_gradient(l, spec, cm);
    *loss = g.loss;
    grads[0] = g.head.x;
    grads[1] = g.head.y;
    for (uint64_t t = 0; t < nn; ++t) {
      grads[2 + 2 * t] = g.neighbors[t].x;
      grads[3 + 2 * t] = g.neighbors[t].y;
    }
    for (uint64_t t = 0; t < s; ++t) {
      grads[2 + 2 * nn + 2 * t] = g.negatives[t].x;
      grads[3 + 2 * nn + 2 * t] = g.negatives[t].y;
    }
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// The epoch loop of fit() (optimizer.hpp:355-470) driven from a given index
// (graph + clusters) and initial layout, calling the reference's own
// build_affinity / shard_clusters / make_noise_model / gather_means /
// lr_schedule / detail::run_worker_epoch. Runs epochs
// [first_epoch, first_epoch + n_run) of a cfg->epochs schedule. The worker RNG
// streams start fresh (as in fit) and are advanced through first_epoch
// skipped epochs only when first_epoch == 0 (callers use first_epoch > 0 only
// for timing). threads: 0 = one std::thread per worker (as fit); 1 = inline.
// seconds_out (nullable): wall time of the epoch loop.
int ref_train_epochs(uint64_t n, uint64_t C, const uint32_t* assign,
                     const uint32_t* offsets, const uint32_t* neighbors,
                     uint64_t k, const ref_train_config* cfgp, double* layout,
                     uint64_t first_epoch, uint64_t n_run, double* epoch_loss,
                     double* final_means, int32_t inline_workers,
                     double* seconds_out) {
  try {
    nomad::TrainConfig cfg;
    cfg.epochs = cfgp->epochs;
    cfg.k = k;
    cfg.negatives = cfgp->negatives;
    cfg.local_draws = cfgp->local_draws;
    cfg.batch_size = cfgp->batch_size;
    cfg.workers = cfgp->workers;
    cfg.seed = cfgp->seed;
    cfg.lr0 = cfgp->lr0;
    cfg.approx = cfgp->approx_all_but_own ? nomad::ApproxMode::AllButOwnCluster
                                          : nomad::ApproxMode::RemoteClusters;
    cfg.head_only = cfgp->head_only != 0;
    cfg.validate();

    nomad::KnnGraph g;
    g.rows = n;
    g.k = k;
    g.offsets.assign(offsets, offsets + n + 1);
    g.neighbors.assign(neighbors, neighbors + offsets[n]);
    g.distances.assign(offsets[n], 0.0);
    auto clusters = make_ca(n, 1, C, assign, nullptr, nullptr);
    const auto affinity = nomad::build_affinity(g);
    const auto plan = nomad::shard_clusters(clusters, cfg.workers);
    const auto noise = nomad::make_noise_model(clusters, cfg.negatives);
    std::vector<uint32_t> owner(n);
    for (uint64_t i = 0; i < n; ++i)
      owner[i] = plan.cluster_to_worker[clusters.assignment[i]];
    const double lr0 = cfg.resolve_lr0(n);

    nomad::LayoutMatrix lay;
    lay.rows = n;
    lay.positions.assign(layout, layout + 2 * n);

    std::vector<nomad::detail::WorkerState> ws(cfg.workers);
    for (uint64_t w = 0; w < cfg.workers; ++w) {
      auto& st = ws[w];
      st.id = static_cast<uint32_t>(w);
      st.points = plan.worker_points[w];
      for (uint32_t i : st.points)
        if (affinity.neighbor_count(i) > 0) st.eligible_heads.push_back(i);
      uint64_t remote = 0;
      for (uint64_t r = 0; r < C; ++r) {
        if (plan.cluster_to_worker[r] == w) continue;
        st.remote_cells.push_back(static_cast<uint32_t>(r));
        st.remote_probs.push_back(noise.cell_probs[r]);
        remote += clusters.sizes[r];
      }
      st.local_mass = static_cast<double>(noise.total - remote) /
                      static_cast<double>(noise.total);
      st.rng = nomad::Rng(nomad::stream_seed(
          cfg.seed, nomad::detail::worker_stream_tag(st.id)));
    }
    std::vector<std::vector<uint32_t>> members;
    if (cfg.approx == nomad::ApproxMode::AllButOwnCluster) {
      members.resize(C);
      for (uint64_t i = 0; i < n; ++i) members[assign[i]].push_back(i);
    }

    auto means = nomad::gather_means(lay, clusters, 0);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t e = first_epoch; e < first_epoch + n_run; ++e) {
      const double lr = nomad::lr_schedule(e, cfg.epochs, lr0);
      const double step = lr / static_cast<double>(cfg.batch_size);
      std::vector<nomad::EpochStats> stats(cfg.workers);
      if (cfg.workers == 1 || inline_workers) {
        for (uint64_t w = 0; w < cfg.workers; ++w)
          stats[w] = nomad::detail::run_worker_epoch(
              lay, affinity, clusters, noise, owner, ws[w], means, step, cfg, e,
              &members);
      } else {
        std::vector<std::thread> pool;
        std::vector<std::string> errs(cfg.workers);
        std::vector<int> kinds(cfg.workers, -1);
        for (uint64_t w = 0; w < cfg.workers; ++w)
          pool.emplace_back([&, w] {
            try {
              stats[w] = nomad::detail::run_worker_epoch(
                  lay, affinity, clusters, noise, owner, ws[w], means, step, cfg,
                  e, &members);
            } catch (const nomad::Error& err) {
              errs[w] = err.what();
              kinds[w] = static_cast<int>(err.kind());
            }
          });
        for (auto& t : pool) t.join();
        for (uint64_t w = 0; w < cfg.workers; ++w)
          if (kinds[w] >= 0)
            throw nomad::Error(static_cast<nomad::ErrorKind>(kinds[w]), errs[w]);
      }
      // optimizer.hpp:414-433 — bit-identical to gather_means (its comment).
      means = nomad::gather_means(lay, clusters, e + 1);
      double loss_sum = 0.0;
      uint64_t heads = 0;
      for (const auto& s : stats) {
        loss_sum += s.loss_sum;
        heads += s.heads;
      }
      if (epoch_loss)
        epoch_loss[e - first_epoch] =
            heads > 0 ? loss_sum / static_cast<double>(heads) : 0.0;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(layout, lay.positions.data(), n * 2 * 8);
    if (final_means) std::memcpy(final_means, means.means.data(), C * 2 * 8);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// metrics.hpp:113-168 / :205-243 — the reference's own quality metrics, used
// only as the checker of final-map quality parity (tests/test_quality_gpu.py).
int ref_neighborhood_preservation(const float* data, uint64_t n, uint64_t d,
                                  const double* layout, uint64_t k, uint64_t sample,
                                  uint64_t seed, double* value, double* std_error) {
  try {
    nomad::LayoutMatrix l;
    l.rows = n;
    l.positions.assign(layout, layout + 2 * n);
    auto r = nomad::neighborhood_preservation(make_ds(data, n, d), l, k, sample, seed);
    *value = r.value;
    *std_error = r.std_error;
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// metrics.hpp:174-200 neighborhood_preservation_ann (graph CSR, layout n x 2)
int ref_neighborhood_preservation_ann(uint64_t n, const uint32_t* offsets,
                                      const uint32_t* neighbors, const double* layout, uint64_t k,
                                      double* value) {
  try {
    nomad::KnnGraph g;
    g.rows = n;
    g.k = k;
    g.offsets.assign(offsets, offsets + n + 1);
    g.neighbors.assign(neighbors, neighbors + offsets[n]);
    g.distances.assign(offsets[n], 0.0);
    nomad::LayoutMatrix l;
    l.rows = n;
    l.positions.assign(layout, layout + 2 * n);
    *value = nomad::neighborhood_preservation_ann(g, l, k).value;
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

int ref_random_triplet_accuracy(const float* data, uint64_t n, uint64_t d,
                                const double* layout, uint64_t count, uint64_t seed,
                                double* value, double* std_error) {
  try {
    nomad::LayoutMatrix l;
    l.rows = n;
    l.positions.assign(layout, layout + 2 * n);
    auto r = nomad::random_triplet_accuracy(make_ds(data, n, d), l, count, seed);
    *value = r.value;
    *std_error = r.std_error;
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// dataset.hpp:223-250 save_layout (ids NULL: "0".."n-1"; labels NULL: none).
int ref_save_layout(const char* path, const double* layout, uint64_t n, const char* const* ids,
                    const char* const* labels) {
  try {
    nomad::LayoutMatrix l;
    l.rows = n;
    l.positions.assign(layout, layout + 2 * n);
    std::vector<std::string> iv(n), lv;
    for (uint64_t i = 0; i < n; ++i) iv[i] = ids ? std::string(ids[i]) : std::to_string(i);
    if (labels)
      for (uint64_t i = 0; i < n; ++i) lv.emplace_back(labels[i]);
    nomad::save_layout(l, iv, lv, path);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// dataset.hpp:122-173 load_vectors_raw (rows / dims 0 = not given); out may
// be NULL (shape only).
int ref_load_vectors_raw(const char* path, uint64_t rows, uint64_t dims, float* out,
                         uint64_t* rows_out, uint64_t* dims_out) {
  try {
    std::optional<std::size_t> r, d;
    if (rows) r = rows;
    if (dims) d = dims;
    auto ds = nomad::load_vectors_raw(path, r, d);
    *rows_out = ds.rows;
    *dims_out = ds.dims;
    if (out) std::memcpy(out, ds.data.data(), ds.data.size() * 4);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

// optimizer.hpp:327-482, the whole pipeline, with the FitReport pieces the
// parity tests need. Pointers are nullable except layout.
int ref_fit(const float* data, uint64_t n, uint64_t d, const ref_train_config* c,
            double* layout, uint32_t* assign, uint64_t* n_clusters_out,
            uint32_t* offsets, uint32_t* neighbors, double* distances,
            double* pca_layout, double* epoch_loss, double* final_means) {
  try {
    nomad::TrainConfig cfg;
    cfg.epochs = c->epochs;
    cfg.k = c->k;
    cfg.negatives = c->negatives;
    cfg.local_draws = c->local_draws;
    cfg.batch_size = c->batch_size;
    cfg.workers = c->workers;
    cfg.n_clusters = c->n_clusters;
    cfg.seed = c->seed;
    cfg.lr0 = c->lr0;
    cfg.kmeans_max_iters = c->kmeans_max_iters;
    cfg.kmeans_tol = c->kmeans_tol;
    cfg.approx = c->approx_all_but_own ? nomad::ApproxMode::AllButOwnCluster
                                       : nomad::ApproxMode::RemoteClusters;
    cfg.head_only = c->head_only != 0;
    nomad::FitReport rep;
    auto l = nomad::fit(make_ds(data, n, d), cfg, &rep);
    std::memcpy(layout, l.positions.data(), n * 2 * 8);
    if (assign) std::memcpy(assign, rep.clusters.assignment.data(), n * 4);
    if (n_clusters_out) *n_clusters_out = rep.clusters.n_clusters;
    if (offsets) std::memcpy(offsets, rep.graph.offsets.data(), (n + 1) * 4);
    if (neighbors)
      std::memcpy(neighbors, rep.graph.neighbors.data(), rep.graph.neighbors.size() * 4);
    if (distances)
      std::memcpy(distances, rep.graph.distances.data(), rep.graph.distances.size() * 8);
    if (pca_layout) std::memcpy(pca_layout, rep.pca.positions.data(), n * 2 * 8);
    if (epoch_loss)
      std::memcpy(epoch_loss, rep.epoch_mean_loss.data(), rep.epoch_mean_loss.size() * 8);
    if (final_means)
      std::memcpy(final_means, rep.final_means.means.data(), rep.final_means.means.size() * 8);
    return 0;
  } catch (const nomad::Error& e) { return fail_code(e); }
}

}  // extern "C"
