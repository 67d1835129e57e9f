/* The boundary from plain C99 (no Python, no torch): include/mlfabric.h + libmlfabric.so.
 * Host-only calls (the planner); prints "C_ABI_OK" when every check passes.
 *
 * mlf_plan: the S:156 SJF instance — sizes {30, 10, 20} MB on one 10 MB/s server down-link
 * -> order (1, 2, 0), commit times 1, 3, 6 s, nothing dropped (tau large).
 * mlf_plan_distribution: one server with a 1 GB/s up-link, one 1 GB request -> T = 1 s.
 * Errors: a null argument -> MLF_E_INVALID with a message in mlf_last_error(). */
#include <stdio.h>
#include <string.h>

#include "mlfabric.h"

#define CHECK(c)                                        \
  do {                                                  \
    if (!(c)) {                                         \
      printf("FAILED: %s (line %d)\n", #c, __LINE__);   \
      return 1;                                         \
    }                                                   \
  } while (0)

int main(void) {
  const int64_t MB = 1000000, S = 1000000000;
  int64_t up[4] = {0, 0, 0, 0}, down[4] = {0, 0, 0, 10 * MB};
  mlf_net net;
  memset(&net, 0, sizeof net);
  net.n_nodes = 4;
  net.nic_up = up;
  net.nic_down = down;
  int32_t node[3] = {0, 1, 2};
  int64_t bytes[3] = {30 * MB, 10 * MB, 20 * MB}, version[3] = {100, 100, 100}, t_avail[3] = {0, 0, 0};
  double norm[3] = {1.0, 1.0, 1.0};
  mlf_batch b = {3, node, bytes, version, t_avail, norm};
  int32_t server[1] = {3};
  mlf_plan_params prm;
  memset(&prm, 0, sizeof prm);
  prm.n_servers = 1;
  prm.server = server;
  prm.v_init = 100;
  prm.tau_max = 10;
  prm.div_max = 0.0;
  int32_t order[3], group[3], cfirst[3], ccount[3], punted[3], gnode[3], rf[3], rc[3], rg[3];
  uint8_t drop[3];
  int64_t ct[3];
  mlf_plan_out out;
  memset(&out, 0, sizeof out);
  out.capacity = 3;
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
  CHECK(mlf_plan(&net, &b, &prm, &out) == MLF_OK);
  CHECK(out.n_commit == 3 && order[0] == 1 && order[1] == 2 && order[2] == 0);
  CHECK(ct[0] == 1 * S && ct[1] == 3 * S && ct[2] == 6 * S);
  CHECK(drop[0] == 0 && drop[1] == 0 && drop[2] == 0);

  int64_t up2[2] = {1000 * MB, 1000 * MB}, down2[2] = {1000 * MB, 1000 * MB};
  mlf_net net2 = {2, up2, down2, NULL, NULL};
  int32_t req[1] = {1}, srv[1] = {0}, dorder[1], dgroup[1];
  int64_t trecv[1], tstart[1];
  mlf_dist_params dp;
  memset(&dp, 0, sizeof dp);
  dp.n_servers = 1;
  dp.server = srv;
  dp.model_bytes = 1000 * MB;
  mlf_dist_out dout;
  memset(&dout, 0, sizeof dout);
  dout.capacity = 1;
  dout.order = dorder;
  dout.group = dgroup;
  dout.t_recv_ns = trecv;
  dout.t_start_ns = tstart;
  CHECK(mlf_plan_distribution(&net2, 1, req, &dp, &dout) == MLF_OK);
  CHECK(dout.t_total_ns == S && trecv[0] == S && tstart[0] == 0 && dgroup[0] == 0);

  CHECK(mlf_plan(NULL, &b, &prm, &out) == MLF_E_INVALID);
  CHECK(strlen(mlf_last_error()) > 0);
  printf("C_ABI_OK\n");
  return 0;
}
