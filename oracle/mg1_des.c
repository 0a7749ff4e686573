/* TEST INFRASTRUCTURE ONLY — M/G/1 discrete-event simulation of the SPRPT-with-limited-
 * preemption rank policy (§3.3 P:394-405 and App. C), used to pin the
 * policy the GPU selection implements against closed forms (tests/test_oracle_mg1.py).
 *
 * Model: one server, Poisson arrivals, job = (x size, r prediction, a age).
 * rank(x,r,a) = r - a   if a < a0 = C*r,   -inf otherwise
 * Lowest rank is served; ties are broken FCFS.  With static predictions and this
 * monotone rank, arrivals and completions are the only decision points (a running job's
 * rank only decreases, waiting jobs' ranks are frozen), so the event loop below is exact.
 * zero_plus = 1 models C -> 0+ (reading D-13): rank r at age 0, -inf once started.
 *
 * Plain C99, no dependencies; built by oracle/mg1.py with gcc -O2 -shared -fPIC.
 * Not shared with, and not linked into, the CUDA library.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct { double rank, arrival; int64_t id; } hkey;

static int hless(const hkey *a, const hkey *b) {
  if (a->rank != b->rank) return a->rank < b->rank;
  if (a->arrival != b->arrival) return a->arrival < b->arrival;
  return a->id < b->id;
}

typedef struct { hkey *v; int64_t n; } heap;

static void hpush(heap *h, hkey k) {
  int64_t i = h->n++;
  h->v[i] = k;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!hless(&h->v[i], &h->v[p])) break;
    hkey t = h->v[i]; h->v[i] = h->v[p]; h->v[p] = t; i = p;
  }
}

static hkey hpop(heap *h) {
  hkey top = h->v[0];
  h->v[0] = h->v[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->n && hless(&h->v[l], &h->v[s])) s = l;
    if (r < h->n && hless(&h->v[r], &h->v[s])) s = r;
    if (s == i) break;
    hkey t = h->v[i]; h->v[i] = h->v[s]; h->v[s] = t; i = s;
  }
  return top;
}

/* rank of job j at age a */
static double rank_of(double r, double a, double C, int zero_plus) {
  if (zero_plus) return a > 0.0 ? -INFINITY : r;
  return (a < C * r) ? r - a : -INFINITY;
}

/* Simulates jobs in arrival order.  arrival[] must be non-decreasing.
 * Outputs: completion[j] (time), first_service[j], preemptions (count),
 * peak_memory = max over time of the sum of ages of started, unfinished jobs (App. D
 * P:946 "memory usage is modeled as proportional to the age of each job").
 * Returns 0 on success, -1 on allocation failure. */
int mg1_simulate(int64_t n, const double *arrival, const double *size, const double *pred,
                 double C, int zero_plus, double *completion, double *first_service,
                 int64_t *preemptions, double *peak_memory) {
  double *age = (double *)calloc((size_t)n, sizeof(double));
  heap h; h.v = (hkey *)malloc(sizeof(hkey) * (size_t)(n + 1)); h.n = 0;
  if (!age || !h.v) { free(age); free(h.v); return -1; }
  for (int64_t j = 0; j < n; ++j) { completion[j] = NAN; first_service[j] = NAN; }
  int64_t cur = -1, next = 0, done = 0, npre = 0;
  double t = 0.0, cur_start = 0.0; /* cur's age at time t = age[cur] + (t - cur_start) */
  double mem_waiting = 0.0, peak = 0.0;   /* sum of ages of started jobs that wait */
  while (done < n) {
    double t_arr = next < n ? arrival[next] : INFINITY;
    double t_cmp = cur >= 0 ? cur_start + (size[cur] - age[cur]) : INFINITY;
    if (cur >= 0) { /* memory just before the next event (max within the interval) */
      double a_end = age[cur] + ((t_arr < t_cmp ? t_arr : t_cmp) - cur_start);
      double mem = mem_waiting + a_end;
      if (mem > peak) peak = mem;
    }
    if (t_cmp <= t_arr) {                 /* completion (ties: complete first) */
      t = t_cmp;
      age[cur] = size[cur];
      completion[cur] = t;
      ++done;
      cur = -1;
      if (h.n > 0) {
        hkey k = hpop(&h);
        cur = k.id; cur_start = t;
        if (age[cur] > 0.0) mem_waiting -= age[cur];
        if (isnan(first_service[cur])) first_service[cur] = t;
      }
    } else {                              /* arrival of job `next` */
      t = t_arr;
      int64_t j = next++;
      if (cur < 0) {
        cur = j; cur_start = t; first_service[j] = t;
      } else {
        age[cur] += t - cur_start; cur_start = t;
        double rc = rank_of(pred[cur], age[cur], C, zero_plus);
        double rj = rank_of(pred[j], 0.0, C, zero_plus);
        if (rj < rc) {                    /* strictly better rank preempts (FCFS on ties) */
          hkey k = { rc, arrival[cur], cur };
          hpush(&h, k);
          mem_waiting += age[cur];
          if (age[cur] > 0.0) ++npre;   /* a zero-age swap is a reorder, not a preemption */
          cur = j; first_service[j] = t;
        } else {
          hkey k = { rj, arrival[j], j };
          hpush(&h, k);
        }
      }
    }
  }
  *preemptions = npre;
  *peak_memory = peak;
  free(age); free(h.v);
  return 0;
}
