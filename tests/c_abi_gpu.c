/* The whole hot path from plain C99 + the CUDA runtime (no Python, no torch):
 * cudaMalloc'd slots and model, mlf_synth_fill inputs (the seeded generator), mlf_init,
 * mlf_submit_update, mlf_batch_view + mlf_plan, mlf_execute, mlf_sync, mlf_pull_model to
 * host memory.  Writes the plan and the pulled model to argv[1] (binary) for
 * tests/test_c_abi.py to check against the oracle.
 *
 * Instance: W = 6 workers on nodes 0..5 with up-links {10, 5, 10, 2.5, 10, 1} MB/s, server
 * node 6 (down-link 10 MB/s), aggregators {0, 2}, tau_max 4, fresh updates (version v0),
 * S = 100003 fp32 elements, lr 0.01, seed 0x4D4C46, iteration 0. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "mlfabric.h"

#define CK(x)                                                                      \
  do {                                                                             \
    if (!(x)) {                                                                    \
      fprintf(stderr, "FAILED %s (line %d): %s\n", #x, __LINE__, mlf_last_error()); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

enum { W = 6, NODES = 7 };

int main(int argc, char **argv) {
  if (argc < 2) return 2;
  const int64_t S = 100003, MB = 1000000;
  const uint64_t seed = 0x4D4C46;
  void *slot[W];
  float *w;
  for (int i = 0; i < W; ++i) CK(cudaMalloc(&slot[i], (size_t)S * 4) == cudaSuccess);
  CK(cudaMalloc((void **)&w, (size_t)S * 4) == cudaSuccess);
  for (int i = 0; i < W; ++i) CK(mlf_synth_fill(0, slot[i], S, 0, MLF_F32, seed, 1, i, 0, 0, NULL) == MLF_OK);
  CK(mlf_synth_fill(0, w, S, 0, MLF_F32, seed, 2, 0, 0, 0, NULL) == MLF_OK);
  CK(cudaDeviceSynchronize() == cudaSuccess);

  int32_t worker_node[W] = {0, 1, 2, 3, 4, 5}, node_rank[NODES] = {0, 0, 0, 0, 0, 0, 0};
  mlf_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.device = 0;
  cfg.world = 1;
  cfg.model_elems = S;
  cfg.shard_elems = S;
  cfg.n_workers = W;
  cfg.update_dtype = MLF_F32;
  cfg.lr = 0.01f;
  cfg.model_shard = w;
  cfg.update_slot = slot;
  cfg.n_nodes = NODES;
  cfg.node_rank = node_rank;
  cfg.worker_node = worker_node;
  mlf_ctx *ctx = NULL;
  const int64_t v0 = 40;
  CK(mlf_init(&cfg, v0, &ctx) == MLF_OK);
  /* worker 0 by mlf_submit_update, the others in one mlf_submit_batch call */
  CK(mlf_submit_update(ctx, 0, v0, 0, 1.0, NULL) == MLF_OK);
  {
    int32_t ws[W - 1];
    int64_t vs[W - 1];
    double ns[W - 1];
    for (int i = 1; i < W; ++i) ws[i - 1] = i, vs[i - 1] = v0, ns[i - 1] = 1.0;
    CK(mlf_submit_batch(ctx, W - 1, ws, vs, NULL, ns) == MLF_OK);
  }

  int64_t up[NODES] = {10 * MB, 5 * MB, 10 * MB, 5 * MB / 2, 10 * MB, 1 * MB, 0};
  int64_t down[NODES] = {0, 0, 0, 0, 0, 0, 10 * MB};
  mlf_net net = {NODES, up, down, NULL, NULL};
  mlf_batch b;
  CK(mlf_batch_view(ctx, &b) == MLF_OK && b.n == W);
  int32_t server[1] = {6}, agg[2] = {0, 2};
  mlf_plan_params prm;
  memset(&prm, 0, sizeof prm);
  prm.n_servers = 1;
  prm.server = server;
  prm.k = 2;
  prm.agg = agg;
  prm.v_init = v0;
  prm.tau_max = 4;
  int32_t order[W], group[W], gnode[W], cfirst[W], ccount[W], punted[W], rf[W], rc[W], rg[W];
  uint8_t drop[W];
  int64_t ct[W];
  mlf_plan_out out;
  memset(&out, 0, sizeof out);
  out.capacity = W;
  out.order = order;
  out.drop_reason = drop;
  out.group = group;
  out.group_node = gnode;
  out.commit_first = cfirst;
  out.commit_count = ccount;
  out.commit_t_ns = ct;
  out.punted = punted;
  out.replica_commit_first = rf;
  out.replica_commit_count = rc;
  out.replica_commit_group = rg;
  CK(mlf_plan(&net, &b, &prm, &out) == MLF_OK);
  CK(mlf_execute(ctx, &out) == MLF_OK);
  float ms = 0.f;
  CK(mlf_sync(ctx, &ms) == MLF_OK);
  float *host = (float *)malloc((size_t)S * 4);
  int64_t version = -1;
  CK(mlf_pull_model(ctx, host, 1, &version) == MLF_OK);
  CK(cudaDeviceSynchronize() == cudaSuccess);
  int64_t kl = 0, h2d = 0, d2h = 0;
  CK(mlf_stats(ctx, &kl, &h2d, &d2h) == MLF_OK);

  FILE *f = fopen(argv[1], "wb");
  CK(f != NULL);
  int32_t hdr[4] = {out.n_commit, out.n_server_commits, (int32_t)(version - v0), (int32_t)kl};
  fwrite(hdr, sizeof hdr, 1, f);
  fwrite(order, sizeof(int32_t), W, f);
  fwrite(drop, 1, W, f);
  fwrite(group, sizeof(int32_t), W, f);
  fwrite(cfirst, sizeof(int32_t), W, f);
  fwrite(ccount, sizeof(int32_t), W, f);
  fwrite(host, 4, (size_t)S, f);
  fclose(f);
  mlf_destroy(ctx);
  for (int i = 0; i < W; ++i) cudaFree(slot[i]);
  cudaFree(w);
  free(host);
  printf("C_GPU_OK commits=%d kernels=%lld\n", out.n_commit, (long long)kl);
  return 0;
}
