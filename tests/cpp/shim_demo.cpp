// Reference-side integration check: the same program calls the reference's
// own header-only functions (nomad::X) and the B200 engine through the shim
// (nomad::b200::X) on identical inputs and compares.
#include <cstdio>
#include <cmath>
#include <cstring>

#include "nomad/nomad.hpp"
#include "nomad_b200/nomad_b200.hpp"

int main() {
  nomad::VectorDataset ds;
  ds.rows = 2000;
  ds.dims = 16;
  nomad::Rng r(42);
  std::vector<double> centres(5 * 16);
  for (double& c : centres) c = 10.0 * r.gaussian();
  for (std::size_t i = 0; i < ds.rows; ++i)
    for (std::size_t j = 0; j < ds.dims; ++j)
      ds.data.push_back(static_cast<float>(centres[(i % 5) * 16 + j] + r.gaussian()));
  int bad = 0;
  auto a = nomad::lsh_init(ds, 6, 3), b = nomad::b200::lsh_init(ds, 6, 3);
  bad += a.assignment != b.assignment || a.centroids != b.centroids;
  const double tol = nomad::default_kmeans_tol(ds);
  bad += tol != nomad::b200::default_kmeans_tol(ds);
  std::vector<double> qa, qb;
  a = nomad::kmeans_em(ds, a, 100, tol, &qa);
  b = nomad::b200::kmeans_em(ds, b, 100, tol, &qb);
  bad += a.assignment != b.assignment || a.centroids != b.centroids || qa != qb;
  auto ga = nomad::build_knn(ds, a, 15), gb = nomad::b200::build_knn(ds, b, 15);
  bad += ga.neighbors != gb.neighbors || ga.distances != gb.distances || ga.offsets != gb.offsets;
  nomad::TrainConfig cfg;
  cfg.epochs = 20;
  cfg.workers = 2;
  cfg.n_clusters = 6;
  cfg.seed = 3;
  nomad::FitReport ra, rb;
  auto la = nomad::fit(ds, cfg, &ra);
  auto lb = nomad::b200::fit(ds, cfg, &rb);
  bad += ra.clusters.assignment != rb.clusters.assignment;
  bad += ra.graph.neighbors != rb.graph.neighbors;
  const double l0 = ra.epoch_mean_loss.back(), l1 = rb.epoch_mean_loss.back();
  // replay mode + bit-exact GPU PCA: the whole fit is bit-identical
  bad += la.positions != lb.positions || ra.epoch_mean_loss != rb.epoch_mean_loss;
  const auto npa = nomad::neighborhood_preservation(ds, la, 10, 500, 1);
  const auto npb = nomad::b200::neighborhood_preservation(ds, la, 10, 500, 1);
  bad += npa.to_json() != npb.to_json();
  const auto ta = nomad::random_triplet_accuracy(ds, la, 20000, 2);
  const auto tb = nomad::b200::random_triplet_accuracy(ds, la, 20000, 2);
  bad += ta.to_json() != tb.to_json();
  std::vector<std::string> ids(ds.rows);
  for (std::size_t i = 0; i < ds.rows; ++i) ids[i] = "row" + std::to_string(i);
  nomad::save_layout(la, ids, {}, "/tmp/shim_demo_ref.csv");
  nomad::b200::save_layout(la, ids, {}, "/tmp/shim_demo_b200.csv");
  {
    std::FILE* f1 = std::fopen("/tmp/shim_demo_ref.csv", "rb");
    std::FILE* f2 = std::fopen("/tmp/shim_demo_b200.csv", "rb");
    int c1 = 0, c2 = 0;
    do {
      c1 = f1 ? std::fgetc(f1) : -2;
      c2 = f2 ? std::fgetc(f2) : -3;
    } while (c1 == c2 && c1 != EOF);
    bad += c1 != c2;
    if (f1) std::fclose(f1);
    if (f2) std::fclose(f2);
  }
  bad += rb.comm.epochs.size() != 20 || rb.comm.epochs[0].size() != 2;
  // every FitReport field from the engine equals the reference's
  bad += ra.affinity.offsets != rb.affinity.offsets || ra.affinity.neighbors != rb.affinity.neighbors ||
         ra.affinity.weights != rb.affinity.weights ||
         ra.affinity.eligible_heads != rb.affinity.eligible_heads;
  bad += ra.plan.cluster_to_worker != rb.plan.cluster_to_worker ||
         ra.plan.worker_clusters != rb.plan.worker_clusters ||
         ra.plan.worker_points != rb.plan.worker_points ||
         ra.plan.worker_point_counts != rb.plan.worker_point_counts;
  bad += ra.pca.positions != rb.pca.positions;
  bad += ra.final_means.means != rb.final_means.means || ra.final_means.counts != rb.final_means.counts ||
         ra.final_means.epoch_stamp != rb.final_means.epoch_stamp;
  for (std::size_t e = 0; e < ra.comm.epochs.size() && e < rb.comm.epochs.size(); ++e)
    for (std::size_t w = 0; w < ra.comm.epochs[e].size() && w < rb.comm.epochs[e].size(); ++w) {
      const auto &x = ra.comm.epochs[e][w], &y = rb.comm.epochs[e][w];
      bad += x.worker != y.worker || x.clusters != y.clusters ||
             x.payload_doubles != y.payload_doubles || x.payload_counts != y.payload_counts;
    }
  const int after_report = bad;
  // TrainConfig{} defaults (auto C = max(ceil(n / 4096), W, 2), 200 epochs)
  {
    nomad::TrainConfig def;
    auto da = nomad::fit(ds, def), db = nomad::b200::fit(ds, def);
    bad += da.positions != db.positions;
  }
  const int after_defaults = bad;
  // the same fit driven over a 2-rank group from this one call (loopback
  // ranks on device 0; distinct devices would be joined by NCCL)
  {
    nomad::b200::options().devices = {0, 0};
    nomad::FitReport rg;
    auto lg = nomad::b200::fit(ds, cfg, &rg);
    nomad::b200::options().devices.clear();
    bad += la.positions != lg.positions || ra.epoch_mean_loss != rg.epoch_mean_loss ||
           ra.final_means.means != rg.final_means.means;
  }
  if (bad) std::fprintf(stderr, "mismatch: report %d defaults %d group %d\n", after_report,
                        after_defaults - after_report, bad - after_defaults);
  try {
    nomad::b200::lsh_init(ds, 1, 0);
    ++bad;
  } catch (const nomad::Error& e) {
    bad += e.kind() != nomad::ErrorKind::Parameter;
  }
  std::printf("%s loss ref %.6f b200 %.6f\n", bad ? "FAIL" : "OK", l0, l1);
  return bad ? 1 : 0;
}
