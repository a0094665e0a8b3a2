// lm_graph.cuh -- the Levenberg-Marquardt loop of lm_solve (lm.py:754-798)
// on the device: the accept/reject decision, the lambda schedule and the
// termination tests run in single-thread kernels that steer conditional graph
// nodes, so a whole solve is ONE graph launch and one read-back at the end
// (the host loop reads two status blocks per LM iteration).
//
//   WHILE (not done) {                              k_lm_tail sets the condition
//     k_lm_head                                     it += 1, IF(linearize) := need_lin
//     IF (need_lin) { linearize; k_lm_gradcheck }   lm.py:758-765
//     k_lm_mid                                      IF(solve) := not done
//     IF (solve) {
//       damped elimination blocks + preconditioner (lambda read on the device)
//       PCG (a nested conditional WHILE node, or the persistent kernel)
//       back-substitution; candidate = post_step(theta + delta); cost(candidate)
//       k_lm_decide                                 lm.py:767-797
//       k_lm_accept                                 theta := candidate if accepted
//     }
//     k_lm_tail                                     it == max_iterations ends the loop
//   }
//
// The decisions are the host loop's (ssfm_lm_solve) expression for
// expression, so the trajectories are identical.
#pragma once
#include "common.cuh"
#include "ssfm.h"

struct LMState {
  // LMConfig (lm.py:36-58)
  double lambda0, lambda_up, lambda_down, lambda_min, lambda_max, rel_cost_tol, grad_tol;
  int max_it, cap;
  // loop state
  double cost, lam, cost_new;
  int it, need_lin, done, term, result, nrec, accepted, fail_status;
  int n_lin, n_solve;            // linearizations and damped solves run (launch accounting)
  long long cg_total;            // CG iterations over all solves
  unsigned long long t_it, t_pcg0, cg_pad_t1;   // iteration start, PCG start / end
  // the failing solve's CG control block (SolverFailure message)
  int fail_iters;
  double fail_rn, fail_tol;
};

struct LMRecDev {
  int iteration, accepted, cg_iters, status;
  double cost_before, cost_after, lam;
  unsigned long long ns, pcg_ns;
};

// status bits -> ssfm_status (status_to_code in ssfm.cu)
__device__ __forceinline__ int lm_status_code(int s) {
  if (s & (ST_SINGULAR_POINT | ST_PIN_POINT | ST_SINGULAR_PRECOND | ST_PIN_RETAINED | ST_PIN_SCALE))
    return SSFM_SINGULAR_BLOCK;
  if (s & (ST_CG_MAXITER | ST_CG_BREAKDOWN)) return SSFM_CG_STALL;
  if (s & ST_ZERO_QUAT) return SSFM_ZERO_QUATERNION;
  if (s & (ST_COMM_TIMEOUT | ST_SCHEDULE)) return SSFM_COMM_ERROR;
  return SSFM_OK;
}

__device__ __forceinline__ unsigned long long lm_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// after the initial cost: the loop state of lm.py:744-752
__global__ void k_lm_init(LMState* s, const double* scal_cost) {
  s->cost = *scal_cost;
  s->lam = s->lambda0;
  s->cost_new = 0.0;
  s->it = 0;
  s->need_lin = 1;
  s->done = s->max_it < 1;
  s->term = SSFM_TERM_MAX_ITER;
  s->result = SSFM_OK;
  s->nrec = 0;
  s->accepted = 0;
  s->fail_status = 0;
  s->n_lin = s->n_solve = 0;
  s->cg_total = 0;
}

__global__ void k_lm_head(LMState* s, cudaGraphConditionalHandle hlin) {
  s->it += 1;
  s->t_it = lm_now();
  s->accepted = 0;
  cudaGraphSetConditional(hlin, s->need_lin ? 1u : 0u);
}

// linearize-time gradient test (lm.py:758-765)
__global__ void k_lm_gradcheck(LMState* s, const double* scal_gmax) {
  s->need_lin = 0;
  s->n_lin += 1;
  if (*scal_gmax < s->grad_tol) {
    s->term = SSFM_TERM_CONVERGED_GRAD;
    s->done = 1;
  }
}

__global__ void k_lm_mid(LMState* s, cudaGraphConditionalHandle hsolve) {
  cudaGraphSetConditional(hsolve, s->done ? 0u : 1u);
}

// accept / reject, lambda schedule, termination (lm.py:767-797)
template <typename Ctl>
__global__ void k_lm_decide(LMState* s, const int* status, const Ctl* ctl, const double* scal_cost,
                            LMRecDev* recs) {
  const unsigned long long now = lm_now();
  const int st = *status;
  const int code = lm_status_code(st);
  const bool pcg_done = !(st & (ST_SINGULAR_POINT | ST_PIN_POINT | ST_SINGULAR_PRECOND | ST_PIN_RETAINED |
                                ST_PIN_SCALE | ST_CG_MAXITER | ST_CG_BREAKDOWN));
  s->n_solve += 1;
  s->cg_total += ctl->iters;
  const bool failed = code != 0;
  s->accepted = 0;
  if (failed && s->lam >= s->lambda_max) {
    s->term = SSFM_TERM_SOLVER_FAILURE;
    s->result = SSFM_SOLVER_FAILURE;
    s->fail_status = st;
    s->fail_iters = ctl->iters;
    s->fail_rn = ctl->rn;
    s->fail_tol = ctl->tol;
    s->done = 1;
    return;
  }
  const double cost_new = failed ? __longlong_as_double(0x7ff8000000000000ll) : *scal_cost;
  const bool accepted = !failed && isfinite(cost_new) && cost_new < s->cost;
  if (s->nrec < s->cap) {
    LMRecDev& R = recs[s->nrec];
    R.iteration = s->it;
    R.cost_before = s->cost;
    R.cost_after = cost_new;
    R.lam = s->lam;
    R.accepted = accepted;
    R.cg_iters = pcg_done ? ctl->iters : 0;
    R.status = code;
    R.ns = now - s->t_it;
    R.pcg_ns = s->cg_pad_t1 >= s->t_pcg0 ? s->cg_pad_t1 - s->t_pcg0 : 0;
  }
  s->nrec += 1;
  if (accepted) {
    const double rel = (s->cost - cost_new) / fmax(s->cost, 1e-300);
    s->cost = cost_new;
    s->lam = fmax(s->lam / s->lambda_down, s->lambda_min);
    s->need_lin = 1;
    s->accepted = 1;
    if (rel < s->rel_cost_tol) {
      s->term = SSFM_TERM_CONVERGED_COST;
      s->done = 1;
    }
  } else {
    s->lam = fmin(s->lam * s->lambda_up, s->lambda_max);
  }
}

// theta := candidate on acceptance (the host loop swaps the two buffers)
__global__ void k_lm_accept(const LMState* s, const double* __restrict__ cand, double* theta, long long n) {
  if (!s->accepted) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    theta[i] = cand[i];
}

__global__ void k_lm_tail(LMState* s, cudaGraphConditionalHandle hwhile) {
  if (!s->done && s->it >= s->max_it) s->done = 1;
  cudaGraphSetConditional(hwhile, s->done ? 0u : 1u);
}
