/* refrun.c -- multi-threaded driver for femopt-emitted element kernels.
 * TEST / BASELINE INFRASTRUCTURE (the reference arm of bench.py).
 *
 * The reference runs an emitted kernel through a uniform pointer-array entry
 * point `kernel_argv(double* const* o, const double* const* t, const double* c)`
 * (proj/tests/test_backend.cpp:62-73,83-98).  The e-loop extent is a literal
 * in the emitted C (emit_c.cpp:95-96), so a kernel emitted with E = chunk is
 * applied to consecutive chunks by offsetting every e-indexed table pointer and
 * every output pointer.  Threads get one contiguous range of
 * chunks each.  Outputs are zeroed per chunk before the
 * call because emitted kernels accumulate with `+=` (emit_c.cpp:129).
 *
 * This file is compiled together with the emitted sources into one shared
 * object by oracle/refkernel.py; nothing here is product code.
 */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef void (*argv_fn)(double* const* o, const double* const* t, const double* c);

typedef struct {
  int nk;
  argv_fn* fns;
  const int *nout, *ntab, *ncon, *idx; /* idx: per kernel [outs..., tabs..., cons...] */
  long chunk;
  double* const* outs;
  const long* out_per_cell;
  const double* const* tabs;
  const int* tab_is_e;
  const double* consts;
  long c0, c1; /* chunk range */
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  double* op[64];
  const double* tp[512];
  double cv[16];
  for (long ch = J->c0; ch < J->c1; ++ch) {
    long e0 = ch * J->chunk;
    const int* ix = J->idx;
    for (int k = 0; k < J->nk; ++k) {
      int no = J->nout[k], nt = J->ntab[k], nc = J->ncon[k];
      for (int i = 0; i < no; ++i) {
        int g = ix[i];
        op[i] = J->outs[g] + e0 * J->out_per_cell[g];
        memset(op[i], 0, sizeof(double) * J->chunk * J->out_per_cell[g]);
      }
      for (int i = 0; i < nt; ++i) {
        int g = ix[no + i];
        tp[i] = J->tabs[g] + (J->tab_is_e[g] ? e0 : 0);
      }
      for (int i = 0; i < nc; ++i) cv[i] = J->consts[ix[no + nt + i]];
      J->fns[k](op, tp, cv);
      ix += no + nt + nc;
    }
  }
  return NULL;
}

/* Runs every kernel over cells [0, E) (E a multiple of `chunk`) on `nthreads`
 * threads.  Returns 0, or -1 on bad arguments. */
int refrun(int nk, void** fns, const int* nout, const int* ntab, const int* ncon, const int* idx,
           long E, long chunk, double* const* outs, const long* out_per_cell,
           const double* const* tabs, const int* tab_is_e, const double* consts, int nthreads) {
  if (chunk <= 0 || E % chunk != 0 || nthreads <= 0 || nthreads > 1024) return -1;
  for (int k = 0; k < nk; ++k)
    if (nout[k] > 64 || ntab[k] > 512 || ncon[k] > 16) return -1;
  long nch = E / chunk;
  if (nthreads > nch) nthreads = (int)(nch > 0 ? nch : 1);
  pthread_t th[1024];
  job_t jobs[1024];
  for (int t = 0; t < nthreads; ++t) {
    job_t* J = &jobs[t];
    J->nk = nk;
    J->fns = (argv_fn*)fns;
    J->nout = nout;
    J->ntab = ntab;
    J->ncon = ncon;
    J->idx = idx;
    J->chunk = chunk;
    J->outs = outs;
    J->out_per_cell = out_per_cell;
    J->tabs = tabs;
    J->tab_is_e = tab_is_e;
    J->consts = consts;
    J->c0 = nch * t / nthreads;
    J->c1 = nch * (t + 1) / nthreads;
    if (t > 0) pthread_create(&th[t], NULL, worker, J);
  }
  worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}
