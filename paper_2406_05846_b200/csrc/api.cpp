// Host-only part of the C-ABI: SDP handles, errors, version, host test hook.
#include <cstring>
#include <new>
#include <string>

#include "host.h"

struct strom_sdp {
  strom::Sdp s;
};

namespace strom {
static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
const Sdp &sdp_of(const strom_sdp *h) { return h->s; }
}  // namespace strom

extern "C" {

const char *strom_last_error(void) { return strom::g_last_error.c_str(); }
const char *strom_version(void) { return "strom-b200 0.1 (sm_100a)"; }

strom_status strom_sdp_create(strom_sdp **out, int32_t nblocks, const strom_block *blocks,
                              int32_t m, const double *b) {
  if (!out) { strom::set_error("strom_sdp_create: out is NULL"); return STROM_EINVAL; }
  *out = nullptr;
  strom_sdp *h = new (std::nothrow) strom_sdp;
  if (!h) { strom::set_error("strom_sdp_create: out of host memory"); return STROM_ENOMEM; }
  strom_status st;
  try {
    st = strom::build_sdp(h->s, nblocks, blocks, m, b);
  } catch (const std::bad_alloc &) {
    st = STROM_ENOMEM;
    strom::set_error("strom_sdp_create: out of host memory");
  }
  if (st != STROM_OK) { delete h; return st; }
  *out = h;
  return STROM_OK;
}

void strom_sdp_destroy(strom_sdp *sdp) { delete sdp; }

strom_status strom_sdp_dims(const strom_sdp *sdp, int64_t *n, int32_t *m, int32_t *nblocks) {
  if (!sdp) { strom::set_error("strom_sdp_dims: NULL handle"); return STROM_EINVAL; }
  if (n) *n = sdp->s.n;
  if (m) *m = sdp->s.m;
  if (nblocks) *nblocks = sdp->s.nblocks;
  return STROM_OK;
}

strom_status strom_debug_host_solve(const strom_sdp *sdp, const strom_admm_config *cfg,
                                    const double *r, double *y) {
  if (!sdp || !cfg || !r || !y) { strom::set_error("strom_debug_host_solve: NULL argument"); return STROM_EINVAL; }
  strom::Factor f;
  strom_status st = strom::build_factor(sdp->s, cfg->eps_rel, cfg->eps, f);
  if (st != STROM_OK) return st;
  st = strom::host_factor_dense(f);
  if (st != STROM_OK) return st;
  strom::host_solve(f, r, y);
  return STROM_OK;
}

strom_status strom_debug_host_part(const strom_sdp *sdp, const strom_admm_config *cfg, int32_t nranks,
                                   int32_t rank, const double *r, double *send, const double *recv,
                                   double *y, int32_t *nB) {
  if (!sdp || !cfg || !r) { strom::set_error("strom_debug_host_part: NULL argument"); return STROM_EINVAL; }
  strom::Factor f;
  strom_status st = strom::build_factor(sdp->s, cfg->eps_rel, cfg->eps, f);
  if (st != STROM_OK) return st;
  strom::PartPlan p;
  if ((st = strom::make_plan(sdp->s, f, nranks, rank, p)) != STROM_OK) return st;
  if (nB) *nB = p.nB;
  if (!send && !(recv && y)) return STROM_OK;
  if ((st = strom::host_factor_dense(f)) != STROM_OK) return st;
  strom::PartFactor pf;
  if ((st = strom::host_factor_partition(f, p, pf)) != STROM_OK) return st;
  if (send) strom::host_part_begin(f, p, pf, r, send);
  if (recv && y) strom::host_part_end(f, p, pf, r, recv, y);
  return STROM_OK;
}

void strom_admm_default_config(strom_admm_config *cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->sigma = 1.0;
  cfg->tau = 1.618;
  cfg->eps_rel = 1e-12;
  cfg->eps = 0.0;
  cfg->sigma_period = 0;
  cfg->sigma_ratio = 2.0;
  cfg->sigma_factor = 1.2;
  cfg->sigma_min = 1e-4;
  cfg->sigma_max = 1e4;
  cfg->check_every = 50;
  cfg->eig_max_sweeps = 40;
  cfg->eig_tol = 1e-15;
  cfg->eig_warm = 1;
  cfg->eig_cold_every = 0;
}

}  // extern "C"
