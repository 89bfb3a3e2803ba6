/*
 * yatt_oracle.c — CPU restatement of the experience-making path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline — never on the product path.
 *
 * Integer path (R1-R6, R10, A5/A6): line-by-line restatement of the
 * reference (/root/reference/proj/...), pinned against the reference itself
 * (oracle/_ref, built by oracle/Makefile from the reference sources) and its
 * known-answer tests — see tests/golden/ and tests/test_oracle_*.py.
 *
 * Float path (A1-A4): the reference has NO implementation of these (SURVEY.md
 * §0.2, §8c).  They are restated here from the standard GRPO / PPO / DAPO
 * definitions, in fp64 with the reference's numerics convention (two-pass
 * max-subtracted softmax, proj/src/distattn.cpp:99-123) and cross-checked
 * against an independent second implementation (torch fp64,
 * tests/test_oracle_float.py).  A1 (logp / ref_logp / entropy / every KL
 * mode) is PINNED to the reference's own fp64 softmax: one
 * distattn::reference_attention head per token row (oracle/softmax_pin.cpp,
 * tests/golden/softmax_pin.json) agrees to 1e-12.  GRPO, GAE and the loss
 * have no reference counterpart at all: "parity unpinned" for A2-A4.
 *
 * Conventions (never changed silently; mirrored in DESIGN.md):
 *   entropy   H = -sum_v p_v log p_v (nats)
 *   KL modes  Delta = ref_logp - logp;  K1 = -Delta, K2 = Delta^2/2,
 *             K3 = exp(Delta) - Delta - 1 (expm1 form), FULL = sum p (log p - log q)
 *   GRPO      group = global sample_id / G; std unbiased (n-1); adv =
 *             (r - mean)/(std + eps) (or r - mean); groups of one -> 0
 *   GAE       masked tokens transparent; V_next = 0 past the end;
 *             A = delta + gamma*lam*A_next; R = A + V
 *   loss      ratio = exp(logp - old); pg = max(-A r, -A clip(r, 1-el, 1+eh));
 *             dual clip for A<0 when c>1; L = pg + kl_coef kl - ent_coef H
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- L0 ---- */
/* proj/include/yatt/common.hpp:17-22 */
uint64_t yo_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
/* common.hpp:25-31 */
uint64_t yo_hash_key(const uint64_t* parts, int n) {
  uint64_t h = 0x243f6a8885a308d3ULL;
  for (int i = 0; i < n; ++i) h = yo_splitmix64(h ^ yo_splitmix64(parts[i]));
  return h;
}
/* common.hpp:35-37 */
double yo_uniform_from_key(uint64_t key) {
  return (double)(yo_splitmix64(key) >> 11) * 0x1.0p-53;
}
static uint64_t hash3(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t p[3] = {a, b, c};
  return yo_hash_key(p, 3);
}
static uint64_t hash5(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e) {
  const uint64_t p[5] = {a, b, c, d, e};
  return yo_hash_key(p, 5);
}

/* ---------------------------------------------------------------- R1 ---- */
/* proj/src/workload.cpp:183-198.  Returns 0 ok, 1 ConfigError, 2 RankOutOfRange */
int yo_shard_dataset(uint64_t total, int p, int r, uint64_t* begin, uint64_t* end) {
  if (p <= 0) return 1;
  if (r < 0 || r >= p) return 2;
  const uint64_t P = (uint64_t)p, R = (uint64_t)r;
  const uint64_t base = total / P, rem = total % P;
  *begin = R * base + (R < rem ? R : rem);
  *end = *begin + base + (R < rem ? 1 : 0);
  return 0;
}

/* ---------------------------------------------------------------- R6 ---- */
/* workload.cpp:15-20 */
static int clamp_length(double value, int max_len) {
  const double rounded = nearbyint(value);
  if (rounded < 1) return 1;
  if (rounded > max_len) return max_len;
  return (int)rounded;
}
/* workload.cpp:23-27 */
static double normal_from_key(uint64_t key) {
  const double two_pi = 6.283185307179586476925286766559;
  const double u1 = yo_uniform_from_key(key);
  const double u2 = yo_uniform_from_key(yo_splitmix64(key ^ 0x5bf0a8b1457e1d23ULL));
  return sqrt(-2.0 * log1p(-u1)) * cos(two_pi * u2);
}
/* workload.cpp:109-132; kind 0 const, 1 uniform, 2 normal, 3 lognormal */
int yo_sample_length_keyed(int kind, double p1, double p2, int max_len, uint64_t seed,
                           uint64_t stream, uint64_t step, uint64_t round, uint64_t id) {
  const uint64_t key = hash5(seed, stream, step, round, id);
  switch (kind) {
    case 0: return clamp_length(p1, max_len);
    case 1: {
      const long long lo = llround(p1), hi = llround(p2);
      const uint64_t span = (uint64_t)(hi - lo) + 1;
      const double u = yo_uniform_from_key(key);
      const long long v = lo + (long long)(u * (double)span);
      return clamp_length((double)v, max_len);
    }
    case 2: return clamp_length(p1 + p2 * normal_from_key(key), max_len);
    default: return clamp_length(exp(p1 + p2 * normal_from_key(key)), max_len);
  }
}

/* Bulk draws for ids id0 .. id0+n-1 (the >= 10^7-draw parity test). */
void yo_sample_lengths_range(int kind, double p1, double p2, int max_len, uint64_t seed,
                             uint64_t stream, uint64_t step, uint64_t round, uint64_t id0,
                             int64_t n, int32_t* out) {
  for (int64_t i = 0; i < n; ++i)
    out[i] = yo_sample_length_keyed(kind, p1, p2, max_len, seed, stream, step, round,
                                    id0 + (uint64_t)i);
}

/* Adversarial keys: ids in [id0, id0+n) whose Normal (kind 2) / LogNormal
 * (kind 3) pre-rounding value v (glibc) lies within band * max(1, |v|) of a
 * .5 rounding tie -- the draws the device cannot certify (keyed_draw.cuh).
 * Returns how many were found; the first `cap` ids go to out. */
int64_t yo_near_ties(int kind, double p1, double p2, uint64_t seed, uint64_t stream,
                     uint64_t step, uint64_t round, uint64_t id0, int64_t n, double band,
                     uint64_t* out, int64_t cap) {
  int64_t found = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t key = hash5(seed, stream, step, round, id0 + (uint64_t)i);
    double v = p1 + p2 * normal_from_key(key);
    if (kind == 3) v = exp(v);
    const double f = v - floor(v);
    if (fabs(f - 0.5) <= band * fmax(1.0, fabs(v))) {
      if (found < cap) out[found] = id0 + (uint64_t)i;
      ++found;
    }
  }
  return found;
}

/* ---------------------------------------------------------------- R5 ---- */
/* workload.cpp:145-167 (validation returns 1 for ConfigError) */
int yo_rejection_flags(const uint64_t* ids, const uint8_t* accepted, int64_t n, int step,
                       int round, double rate, int per_group, int G, uint64_t seed,
                       uint8_t* out) {
  if (rate < 0 || rate >= 1) return 1;
  if (per_group && G <= 0) return 1;
  for (int64_t i = 0; i < n; ++i) {
    out[i] = 0;
    if (accepted[i]) continue;
    const uint64_t unit = per_group ? ids[i] / (uint64_t)G : ids[i];
    out[i] = yo_uniform_from_key(hash5(seed, 3, (uint64_t)(int64_t)step,
                                       (uint64_t)(int64_t)round, unit)) < rate;
  }
  return 0;
}

/* ---------------------------------------------------------------- R3 ---- */
typedef struct {
  uint64_t sample_id;
  int32_t prompt_len_tokens, out_len_tokens, accepted_round, accepted;
} yo_sample;
typedef struct {
  int32_t controller_rank, mb_index, sample_count, max_out_len_tokens;
  int64_t score_tokens;
} yo_mb;
typedef struct {
  int32_t controller_rank, round, active_count, newly_accepted_count, forced_accept_count,
      pending_count;
  int64_t accepted_score_tokens, accepted_train_units, num_microbatches;
} yo_report;

/* simcore.cpp:157-214 with build_microbatches (simcore.cpp:17-39) inlined.
 * mbs must hold ceil(n/mb) entries.  Returns 0 or 1 (ConfigError). */
int yo_shard_round(yo_sample* s, int64_t n, int rank, int step, int round, int kind, double p1,
                   double p2, int max_len, double rate, int per_group, int G, uint64_t seed,
                   int mb, int max_rounds, yo_report* rep, yo_mb* mbs) {
  if (mb <= 0) return 1;
  memset(rep, 0, sizeof(*rep));
  rep->controller_rank = rank;
  rep->round = round;
  int64_t pidx = 0;
  const int final_round = round >= max_rounds;
  for (int64_t i = 0; i < n; ++i) {
    if (s[i].accepted) continue;
    s[i].out_len_tokens = yo_sample_length_keyed(kind, p1, p2, max_len, seed, 2,
                                                 (uint64_t)(int64_t)step, (uint64_t)(int64_t)round,
                                                 s[i].sample_id);
    const int64_t k = pidx / mb;
    if (pidx % mb == 0) {
      mbs[k].controller_rank = rank;
      mbs[k].mb_index = (int32_t)k;
      mbs[k].sample_count = 0;
      mbs[k].max_out_len_tokens = 0;
      mbs[k].score_tokens = 0;
    }
    mbs[k].sample_count += 1;
    if (s[i].out_len_tokens > mbs[k].max_out_len_tokens)
      mbs[k].max_out_len_tokens = s[i].out_len_tokens;
    mbs[k].score_tokens += (int64_t)s[i].prompt_len_tokens + s[i].out_len_tokens;
    ++pidx;
  }
  rep->active_count = (int32_t)pidx;
  rep->num_microbatches = (pidx + mb - 1) / mb;
  for (int64_t i = 0; i < n; ++i) {
    /* second pass over the same pending set (the reference loops `pending`) */
    if (s[i].accepted) continue;
    const uint64_t unit = per_group ? s[i].sample_id / (uint64_t)G : s[i].sample_id;
    const int rej = yo_uniform_from_key(hash5(seed, 3, (uint64_t)(int64_t)step,
                                              (uint64_t)(int64_t)round, unit)) < rate;
    if (rej && !final_round) {
      rep->pending_count++;
      continue;
    }
    if (rej) rep->forced_accept_count++;
    s[i].accepted = 2; /* mark newly accepted; fixed up below */
    s[i].accepted_round = round;
    rep->newly_accepted_count++;
    const long long tok = (long long)s[i].prompt_len_tokens + s[i].out_len_tokens;
    rep->accepted_score_tokens += tok;
    rep->accepted_train_units += tok * tok;
  }
  for (int64_t i = 0; i < n; ++i)
    if (s[i].accepted == 2) s[i].accepted = 1;
  return 0;
}

/* --------------------------------------------------------------- R10 ---- */
/* balancer.cpp:20-25: stable order by length desc, index asc (the bucket
 * shuffle is C++ std::shuffle and is pinned by oracle/_ref instead). */
static const int32_t* g_sort_len;
static int cmp_desc(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (g_sort_len[x] != g_sort_len[y]) return g_sort_len[x] > g_sort_len[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}
void yo_sort_order_desc(const int32_t* len, int64_t n, uint32_t* order) {
  for (int64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  g_sort_len = len;
  qsort(order, (size_t)n, sizeof(uint32_t), cmp_desc);
}
/* balancer.cpp:43-56 over a flat bucket list */
double yo_padding_waste(const uint32_t* flat, const int64_t* off, int64_t nb, const int32_t* len) {
  double real = 0, padded = 0;
  for (int64_t b = 0; b < nb; ++b) {
    int mx = 0;
    for (int64_t i = off[b]; i < off[b + 1]; ++i) {
      const int l = len[flat[i]];
      if (l > mx) mx = l;
      real += (double)l * l;
    }
    padded += (double)(off[b + 1] - off[b]) * ((double)mx * mx);
  }
  return padded == 0 ? 0 : 1.0 - real / padded;
}

/* -------------------------------------------------------- synthetic ---- */
static uint16_t bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float bf16_to_f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
/* Same recipe as paper_2508_07970_b200/csrc/synth.cu. */
void yo_synth_logits(uint64_t seed, int64_t row0, int64_t rows, int32_t V, uint16_t* pol,
                     uint16_t* ref, int32_t* tgt) {
  for (int64_t r = 0; r < rows; ++r) {
    const uint64_t g = (uint64_t)(row0 + r);
    const int32_t y = (int32_t)(yo_splitmix64(hash3(seed, 103, g)) % (uint64_t)V);
    tgt[r] = y;
    const uint64_t rk = hash3(seed, 101, g);
    for (int32_t v = 0; v < V; ++v) {
      const uint64_t h = yo_splitmix64(rk + (uint64_t)v);
      const float x = (float)((int)(h >> 56) - 128) * (1.0f / 16.0f);
      float d;
      if (v == y) {
        const int mag = 8 + (int)((h >> 48) & 7);
        d = (float)(((h >> 47) & 1) ? mag : -mag) * (1.0f / 32.0f);
      } else {
        d = (float)((int)((h >> 48) & 31) - 16) * (1.0f / 32.0f);
      }
      pol[r * (int64_t)V + v] = bf16_rne(x);
      ref[r * (int64_t)V + v] = bf16_rne(x + d);
    }
  }
}
void yo_synth_floats(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n, int kind, int G,
                     const float* base, float* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t gi = (uint64_t)(i0 + i);
    const uint64_t key = hash3(seed, stream_id, gi);
    const uint64_t h = yo_splitmix64(key);
    float v = 0.f;
    switch (kind) {
      case 0: v = -(float)(h >> 54) * (1.0f / 64.0f); break;
      case 1: v = (base ? base[i] : 0.f) + (float)((int)(h >> 57) - 64) * (1.0f / 256.0f); break;
      case 2: v = (float)((int)(h >> 56) - 128) * (1.0f / 64.0f); break;
      case 3: v = (float)(h >> 56) * (1.0f / 1024.0f); break;
      case 4: v = (float)((int)(h >> 53) - 1024) * (1.0f / 1024.0f); break;
      case 5: {
        const uint64_t g = gi / (uint64_t)G;
        const uint64_t sel = yo_splitmix64(hash3(seed, stream_id + 1000, g)) & 3;
        const double pg = sel == 0 ? 0.0 : sel == 1 ? 1.0 : sel == 2 ? 0.5
                        : yo_uniform_from_key(hash3(seed, stream_id + 2000, g));
        v = yo_uniform_from_key(key) < pg ? 1.0f : 0.0f;
        break;
      }
      default: break;
    }
    out[i] = v;
  }
}

/* ---------------------------------------------------------------- A1 ---- */
typedef struct {
  const uint16_t *pol, *ref;
  const int32_t* tgt;
  const uint8_t* mask;
  int64_t r0, r1;
  int32_t V, kl_mode;
  double *logp, *ref_logp, *ent, *kl;
} a1_job;

/* Two-pass max-subtracted log-softmax in fp64 (distattn.cpp:99-123 pattern). */
static void a1_rows(const a1_job* j) {
  const int32_t V = j->V;
  for (int64_t r = j->r0; r < j->r1; ++r) {
    if (j->mask && !j->mask[r]) {
      j->logp[r] = j->ref_logp[r] = j->ent[r] = j->kl[r] = 0.0;
      continue;
    }
    const uint16_t* x = j->pol + r * (int64_t)V;
    const uint16_t* z = j->ref + r * (int64_t)V;
    double mx = -INFINITY, mz = -INFINITY;
    for (int32_t v = 0; v < V; ++v) {
      const double a = bf16_to_f(x[v]), b = bf16_to_f(z[v]);
      if (a > mx) mx = a;
      if (b > mz) mz = b;
    }
    double sx = 0, sz = 0, sxx = 0;
    for (int32_t v = 0; v < V; ++v) {
      const double a = bf16_to_f(x[v]) - mx;
      const double e = exp(a);
      sx += e;
      if (e > 0) sxx += e * a; /* 0 * (-inf) contributes nothing */
      sz += exp(bf16_to_f(z[v]) - mz);
    }
    const double lse_p = mx + log(sx), lse_q = mz + log(sz);
    const int32_t y = j->tgt[r];
    const double logp = bf16_to_f(x[y]) - lse_p;
    const double rlogp = bf16_to_f(z[y]) - lse_q;
    j->logp[r] = logp;
    j->ref_logp[r] = rlogp;
    j->ent[r] = log(sx) - sxx / sx; /* H = lse - E_p[x] with x shifted by mx */
    const double delta = rlogp - logp;
    double kl;
    switch (j->kl_mode) {
      case 0: kl = -delta; break;
      case 1: kl = 0.5 * delta * delta; break;
      case 2: kl = expm1(delta) - delta; break;
      default: {
        double acc = 0;
        for (int32_t v = 0; v < V; ++v) {
          const double lp = bf16_to_f(x[v]) - lse_p, lq = bf16_to_f(z[v]) - lse_q;
          if (lp > -INFINITY) acc += exp(lp) * (lp - lq);
        }
        kl = acc;
      }
    }
    j->kl[r] = kl;
  }
}
static void* a1_thread(void* arg) {
  a1_rows((const a1_job*)arg);
  return NULL;
}
/* Multi-threaded over rows (nthreads <= 256). */
void yo_token_stats(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                    const uint8_t* mask, int64_t rows, int32_t V, int32_t kl_mode, double* logp,
                    double* ref_logp, double* ent, double* kl, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads > rows) nthreads = rows > 0 ? (int)rows : 1;
  pthread_t th[256];
  a1_job jobs[256];
  const int64_t per = (rows + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    a1_job jb = {pol, ref, tgt, mask, t * per, (t + 1) * per < rows ? (t + 1) * per : rows,
                 V, kl_mode, logp, ref_logp, ent, kl};
    jobs[t] = jb;
    if (jobs[t].r0 > jobs[t].r1) jobs[t].r0 = jobs[t].r1;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, a1_thread, &jobs[t]);
  a1_rows(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- A2 ---- */
void yo_grpo_advantages(const float* r, int64_t n, uint64_t first_id, int G, float eps,
                        int norm_by_std, double* adv) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t g = (first_id + (uint64_t)i) / (uint64_t)G;
    int64_t lo = (int64_t)(g * (uint64_t)G) - (int64_t)first_id;
    int64_t hi = (int64_t)((g + 1) * (uint64_t)G) - (int64_t)first_id;
    if (lo < 0) lo = 0;
    if (hi > n) hi = n;
    const double cnt = (double)(hi - lo);
    double sum = 0, m2 = 0;
    for (int64_t k = lo; k < hi; ++k) sum += r[k];
    const double mean = sum / cnt;
    for (int64_t k = lo; k < hi; ++k) m2 += (r[k] - mean) * (r[k] - mean);
    double a = 0;
    if (cnt > 1) {
      const double c = (double)r[i] - mean;
      a = norm_by_std ? c / (sqrt(m2 / (cnt - 1)) + (double)eps) : c;
    }
    adv[i] = a;
  }
}

/* ---------------------------------------------------------------- A3 ---- */
void yo_gae(const float* values, const float* rewards, const uint8_t* mask, const int64_t* cu,
            int64_t nseq, double gamma, double lam, double* adv, double* ret) {
  for (int64_t s = 0; s < nseq; ++s) {
    double A = 0, Vn = 0;
    for (int64_t t = cu[s + 1] - 1; t >= cu[s]; --t) {
      const double v = values[t];
      if (!mask || mask[t]) {
        const double delta = (double)rewards[t] + gamma * Vn - v;
        A = delta + gamma * lam * A;
        Vn = v;
      }
      adv[t] = A;
      ret[t] = A + v;
    }
  }
}
void yo_masked_moments(const double* x, const uint8_t* mask, int64_t n, double* out) {
  double c = 0, s = 0, q = 0;
  for (int64_t i = 0; i < n; ++i)
    if (!mask || mask[i]) {
      c += 1;
      s += x[i];
      q += x[i] * x[i];
    }
  out[0] = c;
  out[1] = s;
  out[2] = q;
}

/* ---------------------------------------------------------------- A4 ---- */
/* sums: loss, pg, kl, ent, clip, ratio, tokens, seqs (yatt_loss_sums order) */
void yo_policy_loss(const float* logp, const float* old_logp, const float* adv, const float* kl,
                    const float* ent, const uint8_t* mask, int64_t n, const int64_t* cu,
                    int64_t nseq, float clip_low, float clip_high, float clip_c, float kl_coef,
                    float ent_coef, int agg_mode, double* sums) {
  for (int f = 0; f < 8; ++f) sums[f] = 0;
  const int64_t nsq = agg_mode == 0 ? 1 : nseq;
  for (int64_t s = 0; s < nsq; ++s) {
    const int64_t b = agg_mode == 0 ? 0 : cu[s], e = agg_mode == 0 ? n : cu[s + 1];
    double sl = 0, cnt = 0;
    for (int64_t i = b; i < e; ++i) {
      if (mask && !mask[i]) continue;
      const double ratio = exp((double)logp[i] - (double)old_logp[i]);
      const double a = adv[i];
      const double pg1 = -a * ratio;
      double cl = ratio;
      if (cl < 1.0 - (double)clip_low) cl = 1.0 - (double)clip_low;
      if (cl > 1.0 + (double)clip_high) cl = 1.0 + (double)clip_high;
      const double pg2 = -a * cl;
      double pg = pg1 > pg2 ? pg1 : pg2;
      if (clip_c > 1.f && a < 0) {
        const double p3 = -a * (double)clip_c;
        if (p3 < pg) pg = p3;
      }
      const double k = kl ? kl[i] : 0.0, h = ent ? ent[i] : 0.0;
      sl += pg + (double)kl_coef * k - (double)ent_coef * h;
      sums[1] += pg;
      sums[2] += k;
      sums[3] += h;
      sums[4] += pg2 > pg1;
      sums[5] += ratio;
      cnt += 1;
    }
    if (agg_mode == 0) {
      sums[0] = sl;
      sums[6] = cnt;
    } else if (cnt > 0) {
      sums[0] += agg_mode == 1 ? sl / cnt : sl;
      sums[6] += cnt;
      sums[7] += 1;
    }
  }
}

/* ------------------------------------------------------------- A5/A6 ---- */
/* Returns kept samples; counts[3] = {samples, tokens, groups}.  Group of    */
/* sample i is i / G (workload.cpp:158-160); a trailing partial group (n not  */
/* a multiple of G) is a group of its own, keep has ceil(n / G) entries.      */
int64_t yo_filter_compact(const float* r, const int64_t* lens, int64_t n, int G, uint8_t* keep,
                          int32_t* map, int64_t* new_cu, int64_t* counts) {
  int64_t j = 0, tok = 0, kg = 0;
  for (int64_t g = 0; g < (n + G - 1) / G; ++g) {
    uint32_t b0;
    memcpy(&b0, &r[g * G], 4);
    uint8_t k = 0;
    const int64_t m = n - g * G < G ? n - g * G : G;
    for (int64_t i = 1; i < m; ++i) {
      uint32_t bi;
      memcpy(&bi, &r[g * G + i], 4);
      k |= bi != b0;
    }
    keep[g] = k;
    kg += k;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (!keep[i / G]) continue;
    map[j] = (int32_t)i;
    new_cu[j] = tok;
    tok += lens[i];
    ++j;
  }
  new_cu[j] = tok;
  counts[0] = j;
  counts[1] = tok;
  counts[2] = kg;
  return j;
}

/* ------------------------------------------------------- backward (8f#1) */
/* dL/dx for the policy loss of yo_policy_loss (same config), fp64, from the
 * logits with exact two-pass softmaxes.  Per-token inputs (logp, ref_logp,
 * old_logp, adv) are the fp32 arrays the device also consumes, so clip
 * decisions match.  norm: global token count (agg 0) or seq count (1, 2). */
void yo_logits_backward(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                        const uint8_t* mask, int64_t rows, int32_t V, const float* logp,
                        const float* ref_logp, const float* old_logp, const float* adv,
                        const int64_t* cu, int64_t nseq, float clip_low, float clip_high,
                        float clip_c, float kl_coef, float ent_coef, int agg_mode, int kl_mode,
                        double norm, double* grad, double* coef_out) {
  for (int64_t r = 0; r < rows; ++r) {
    double* gr = grad + r * (int64_t)V;
    if (mask && !mask[r]) {
      for (int32_t v = 0; v < V; ++v) gr[v] = 0;
      continue;
    }
    double scale = 1.0 / norm;
    if (agg_mode == 1) {
      int64_t s = 0;
      while (!(cu[s] <= r && r < cu[s + 1])) ++s;
      double cnt = 0;
      for (int64_t i = cu[s]; i < cu[s + 1]; ++i) cnt += (!mask || mask[i]);
      scale /= cnt;
    }
    const double lp = logp[r], A = adv[r];
    const double ratio = exp(lp - (double)old_logp[r]);
    const double pg1 = -A * ratio;
    double cl = ratio;
    if (cl < 1.0 - (double)clip_low) cl = 1.0 - (double)clip_low;
    if (cl > 1.0 + (double)clip_high) cl = 1.0 + (double)clip_high;
    const double pg2 = -A * cl;
    const double pg = pg1 > pg2 ? pg1 : pg2;
    int active = !(pg2 > pg1);
    if (clip_c > 1.f && A < 0 && -A * (double)clip_c < pg) active = 0;
    const double dpg = active ? -A * ratio : 0.0;
    const double rl = ref_logp ? (double)ref_logp[r] : lp;
    double dkl = 0;
    if (kl_mode == 0) dkl = 1.0;
    else if (kl_mode == 1) dkl = lp - rl;
    else if (kl_mode == 2) dkl = -expm1(rl - lp);
    const double g = scale * (dpg + (kl_mode == 3 ? 0.0 : (double)kl_coef * dkl));
    const double h = scale * (double)ent_coef;
    const double f = kl_mode == 3 ? scale * (double)kl_coef : 0.0;
    const uint16_t* x = pol + r * (int64_t)V;
    const uint16_t* z = ref ? ref + r * (int64_t)V : NULL;
    double mx = -INFINITY, mz = -INFINITY;
    for (int32_t v = 0; v < V; ++v) {
      const double a = bf16_to_f(x[v]);
      if (a > mx) mx = a;
      if (z) {
        const double b = bf16_to_f(z[v]);
        if (b > mz) mz = b;
      }
    }
    double sx = 0, sz = 0;
    for (int32_t v = 0; v < V; ++v) {
      sx += exp(bf16_to_f(x[v]) - mx);
      if (z) sz += exp(bf16_to_f(z[v]) - mz);
    }
    const double lse = mx + log(sx), lseq = z ? mz + log(sz) : 0.0;
    double H = 0, KL = 0;
    for (int32_t v = 0; v < V; ++v) {
      const double lpv = bf16_to_f(x[v]) - lse;
      const double pv = exp(lpv);
      if (pv > 0) H -= pv * lpv;
      if (z && pv > 0) KL += pv * (lpv - (bf16_to_f(z[v]) - lseq));
    }
    for (int32_t v = 0; v < V; ++v) {
      const double lpv = bf16_to_f(x[v]) - lse;
      const double pv = exp(lpv);
      double val = g * ((v == tgt[r]) - pv) + h * pv * (lpv + H);
      if (f != 0) val += f * pv * (lpv - (bf16_to_f(z[v]) - lseq) - KL);
      gr[v] = val;
    }
    if (coef_out) {
      coef_out[4 * r + 0] = g;
      coef_out[4 * r + 1] = h;
      coef_out[4 * r + 2] = f;
      coef_out[4 * r + 3] = lse;
    }
  }
}
