// oracle/oracle.cpp -- fp64 CPU oracle for the GESR MoA candidate-scoring hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code,
// header, table or helper with the CUDA path (paper_2511_21095_b200/csrc) and the
// CUDA path never includes or links it.
//
// Everything here is the plain definition of what the paper computes, written out
// in fp64 with no blocking, fusion or reordering beyond the definition:
//
//   oracle_kv_project       K = act(U W_k^T + b_k), V = act(U W_v^T + b_v), per head
//                           PAPER.md:335-341 (s3.4.2: U in R^{N x D}, D flattened over heads;
//                           the [U,T] self-attention layer's projections applied to U rows).
//                           Projection form act(XW^T+b), act in {identity, SiLU}: SPEC.md:343
//                           (reading R3).
//   oracle_tasa_score       candidate rows I_NRO of one masked self-attention layer over
//                           [U,T]: each candidate attends to all L_b history keys and to no
//                           other candidate.  PAPER.md:341 (mask rules 1-2)
//                           (T_self = HSTU([U,T])[I_NRO]); softmax normalisation with max
//                           subtraction SPEC.md:67, 343 (readings R1, R2, R4-R6).
//   oracle_full_masked_attention
//                           brute force: builds the (L+C)x(L+C) mask from the rules
//                           (SPEC.md:277, 295-297), projects every row of [U;T]
//                           and runs plain masked softmax attention for every row.
//   oracle_build_mask       the mask alone (SPEC.md:289-297 examples are golden fixtures).
//   oracle_hma_count        c = sum_i sum_j [u_i == t_j], then min(c, M) if M > 0.
//                           PAPER.md:308-312 (s3.4.1: binary attention matrix summed against
//                           a value tensor of ones; cap M).  SPEC.md:215-223.
//   oracle_hma_count_hash   a second, independent algorithm for the same count
//                           (multiplicity hash map); used only to cross-check.
//
// bf16 inputs arrive as raw uint16 bit patterns and are widened exactly to double.
// Threads: std::thread over rows / candidates; results do not depend on thread count.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <unordered_map>
#include <vector>
#include <algorithm>

namespace {

double widen_bf16(uint16_t bits) {
  uint32_t u = static_cast<uint32_t>(bits) << 16;
  float f;
  std::memcpy(&f, &u, sizeof(f));
  return static_cast<double>(f);
}

// Round a double to the nearest bf16 value (ties to even), returned as double.
// Used only by the diagnostic rounding-aware mode (reading R8).
double round_to_bf16(double x) {
  float f = static_cast<float>(x);  // double -> float is RNE
  uint32_t u;
  std::memcpy(&u, &f, sizeof(u));
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<double>(f);  // inf / nan
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  u &= 0xffff0000u;
  std::memcpy(&f, &u, sizeof(f));
  return static_cast<double>(f);
}

// act(x): 0 = identity, 1 = SiLU x / (1 + e^-x)
double act_apply(int act, double x) {
  if (act == 1) return x / (1.0 + std::exp(-x));
  return x;
}

template <class F>
void parallel_for(int64_t n, int threads, F&& body) {
  if (n <= 0) return;
  if (threads < 1) threads = 1;
  if (threads > n) threads = static_cast<int>(n);
  if (threads == 1) {
    for (int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads);
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (int64_t i = t; i < n; i += threads) body(i);
    });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int oracle_version(void) { return 1; }

void oracle_round_to_bf16(double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] = round_to_bf16(x[i]);
}

// K[h][r][j] = act( sum_k U[r][k] * W_k[h*d+j][k] + b_k[h*d+j] ), likewise V.
// U: bf16 bits [total_L, D_in]; W_k, W_v: bf16 bits [H*d, D_in]; b_k, b_v: fp64 [H*d] or NULL.
// K, V: fp64 [H, total_L, d] (written).
void oracle_kv_project(const uint16_t* U, int64_t total_L, int32_t D_in,
                       const uint16_t* W_k, const uint16_t* W_v,
                       const double* b_k, const double* b_v,
                       int32_t H, int32_t d, int32_t act,
                       double* K, double* V, int32_t threads) {
  const int64_t HD = static_cast<int64_t>(H) * d;
  parallel_for(total_L, threads, [&](int64_t r) {
    std::vector<double> u(D_in);
    for (int32_t k = 0; k < D_in; ++k) u[k] = widen_bf16(U[r * D_in + k]);
    for (int64_t n = 0; n < HD; ++n) {
      double sk = 0.0, sv = 0.0;
      for (int32_t k = 0; k < D_in; ++k) {
        sk += u[k] * widen_bf16(W_k[n * D_in + k]);
        sv += u[k] * widen_bf16(W_v[n * D_in + k]);
      }
      if (b_k) sk += b_k[n];
      if (b_v) sv += b_v[n];
      const int64_t h = n / d, j = n % d;
      K[(h * total_L + r) * d + j] = act_apply(act, sk);
      V[(h * total_L + r) * d + j] = act_apply(act, sv);
    }
  });
}

// For request b, candidate t in [cand_offsets[b], cand_offsets[b+1]), head h:
//   q    = act(T[t] W_q^T + b_q)[h*d : (h+1)*d]
//   s_i  = scale * sum_j q_j K[h][r_i][j],   r_i in [seq_offsets[b], seq_offsets[b+1])
//   m    = max_i s_i ;  w_i = exp(s_i - m)
//   O[t][h*d + j] = sum_i w_i V[h][r_i][j] / sum_i w_i ;  lse[t][h] = m + log sum_i w_i
//   L_b = 0: O row = 0, lse = -inf  (reading R6)
// round_q_bf16 != 0 rounds q to bf16 before use (diagnostic rounding-aware mode only).
// lse may be NULL.
void oracle_tasa_score(const uint16_t* T, int64_t total_C, int32_t D_in,
                       const int64_t* cand_offsets,
                       const uint16_t* W_q, const double* b_q, int32_t act,
                       const double* K, const double* V,
                       const int64_t* seq_offsets, int64_t B, int64_t total_L,
                       int32_t H, int32_t d, double scale, int32_t round_q_bf16,
                       double* O, double* lse, int32_t threads) {
  const int64_t HD = static_cast<int64_t>(H) * d;
  // candidate -> request map (plain walk over the offsets)
  std::vector<int64_t> owner(total_C, -1);
  for (int64_t b = 0; b < B; ++b)
    for (int64_t t = cand_offsets[b]; t < cand_offsets[b + 1]; ++t) owner[t] = b;
  parallel_for(total_C, threads, [&](int64_t t) {
    const int64_t b = owner[t];
    if (b < 0) return;
    const int64_t r0 = seq_offsets[b], r1 = seq_offsets[b + 1];
    const int64_t Lb = r1 - r0;
    std::vector<double> x(D_in), q(HD), s(Lb > 0 ? Lb : 1);
    for (int32_t k = 0; k < D_in; ++k) x[k] = widen_bf16(T[t * D_in + k]);
    for (int64_t n = 0; n < HD; ++n) {
      double acc = 0.0;
      for (int32_t k = 0; k < D_in; ++k) acc += x[k] * widen_bf16(W_q[n * D_in + k]);
      if (b_q) acc += b_q[n];
      q[n] = act_apply(act, acc);
      if (round_q_bf16) q[n] = round_to_bf16(q[n]);
    }
    for (int32_t h = 0; h < H; ++h) {
      double* o = O + t * HD + static_cast<int64_t>(h) * d;
      if (Lb == 0) {
        for (int32_t j = 0; j < d; ++j) o[j] = 0.0;
        if (lse) lse[t * H + h] = -std::numeric_limits<double>::infinity();
        continue;
      }
      double m = -std::numeric_limits<double>::infinity();
      for (int64_t i = 0; i < Lb; ++i) {
        const double* kr = K + (static_cast<int64_t>(h) * total_L + r0 + i) * d;
        double acc = 0.0;
        for (int32_t j = 0; j < d; ++j) acc += q[static_cast<int64_t>(h) * d + j] * kr[j];
        s[i] = scale * acc;
        m = std::max(m, s[i]);
      }
      double denom = 0.0;
      std::vector<double> num(d, 0.0);
      for (int64_t i = 0; i < Lb; ++i) {
        const double w = std::exp(s[i] - m);
        denom += w;
        const double* vr = V + (static_cast<int64_t>(h) * total_L + r0 + i) * d;
        for (int32_t j = 0; j < d; ++j) num[j] += w * vr[j];
      }
      for (int32_t j = 0; j < d; ++j) o[j] = num[j] / denom;
      if (lse) lse[t * H + h] = m + std::log(denom);
    }
  });
}

// Target-aware mask over [U, T] (N = L history rows, n = C candidate rows), true = may attend.
// The four rules (PAPER.md:341 rules 1-2; SPEC.md:277 adds U-not-to-T and the candidate
// diagonal; self_key selects whether the diagonal is on -- DESIGN.md reading R2):
//   i <  N, j <  N : j <= i          (history is causal)
//   i <  N, j >= N : false           (history never sees candidates)
//   i >= N, j <  N : true            (a candidate sees the whole history)
//   i >= N, j >= N : self_key && i == j   (candidates never see one another)
void oracle_build_mask(int64_t N, int64_t n, int32_t self_key, uint8_t* mask) {
  const int64_t S = N + n;
  for (int64_t i = 0; i < S; ++i) {
    for (int64_t j = 0; j < S; ++j) {
      bool allowed;
      if (i < N && j < N) allowed = (j <= i);
      else if (i < N && j >= N) allowed = false;
      else if (i >= N && j < N) allowed = true;
      else allowed = (self_key != 0) && (i == j);
      mask[i * S + j] = allowed ? 1 : 0;
    }
  }
}

// Brute force for ONE request: X = [U; T] ((L+C) x D_in); Q/K/V = act(X W^T + b) for every
// row; masked softmax attention for every row with at least one allowed key; returns the C
// candidate rows in O_cand [C, H*d] and their lse [C, H] (lse may be NULL).  Rows with no
// allowed key (a candidate with L = 0 and the diagonal off) are 0 / -inf.
void oracle_full_masked_attention(const uint16_t* U, int64_t L, const uint16_t* T, int64_t C,
                                  int32_t D_in,
                                  const uint16_t* W_q, const uint16_t* W_k, const uint16_t* W_v,
                                  const double* b_q, const double* b_k, const double* b_v,
                                  int32_t H, int32_t d, int32_t act, double scale,
                                  int32_t self_key, double* O_cand, double* lse_cand) {
  const int64_t S = L + C;
  const int64_t HD = static_cast<int64_t>(H) * d;
  std::vector<double> X(S * D_in);
  for (int64_t i = 0; i < L; ++i)
    for (int32_t k = 0; k < D_in; ++k) X[i * D_in + k] = widen_bf16(U[i * D_in + k]);
  for (int64_t i = 0; i < C; ++i)
    for (int32_t k = 0; k < D_in; ++k) X[(L + i) * D_in + k] = widen_bf16(T[i * D_in + k]);
  auto project = [&](const uint16_t* W, const double* bias, std::vector<double>& Y) {
    Y.assign(S * HD, 0.0);
    for (int64_t i = 0; i < S; ++i)
      for (int64_t n = 0; n < HD; ++n) {
        double acc = 0.0;
        for (int32_t k = 0; k < D_in; ++k) acc += X[i * D_in + k] * widen_bf16(W[n * D_in + k]);
        if (bias) acc += bias[n];
        Y[i * HD + n] = act_apply(act, acc);
      }
  };
  std::vector<double> Qa, Ka, Va;
  project(W_q, b_q, Qa);
  project(W_k, b_k, Ka);
  project(W_v, b_v, Va);
  std::vector<uint8_t> mask(S * S);
  oracle_build_mask(L, C, self_key, mask.data());
  for (int64_t c = 0; c < C; ++c) {
    const int64_t i = L + c;
    for (int32_t h = 0; h < H; ++h) {
      std::vector<double> sc;
      std::vector<int64_t> idx;
      for (int64_t j = 0; j < S; ++j) {
        if (!mask[i * S + j]) continue;
        double acc = 0.0;
        for (int32_t e = 0; e < d; ++e) acc += Qa[i * HD + h * d + e] * Ka[j * HD + h * d + e];
        sc.push_back(scale * acc);
        idx.push_back(j);
      }
      double* o = O_cand + c * HD + static_cast<int64_t>(h) * d;
      if (sc.empty()) {
        for (int32_t e = 0; e < d; ++e) o[e] = 0.0;
        if (lse_cand) lse_cand[c * H + h] = -std::numeric_limits<double>::infinity();
        continue;
      }
      const double m = *std::max_element(sc.begin(), sc.end());
      double denom = 0.0;
      for (double v : sc) denom += std::exp(v - m);
      for (int32_t e = 0; e < d; ++e) {
        double acc = 0.0;
        for (size_t z = 0; z < sc.size(); ++z)
          acc += std::exp(sc[z] - m) / denom * Va[idx[z] * HD + h * d + e];
        o[e] = acc;
      }
      if (lse_cand) lse_cand[c * H + h] = m + std::log(denom);
    }
  }
}

// counts[t*F + f] = sum_{i in user segment b*F+f} sum_{j in item segment t*F+f} [u_i == t_j],
// b the request owning candidate t; then min(count, cap) if cap > 0.
void oracle_hma_count(const int64_t* user_ids, const int64_t* user_offsets,
                      const int64_t* item_ids, const int64_t* item_offsets,
                      const int64_t* cand_offsets, int64_t B, int64_t total_C, int32_t F,
                      int32_t cap, int32_t* counts, int32_t threads) {
  std::vector<int64_t> owner(total_C, -1);
  for (int64_t b = 0; b < B; ++b)
    for (int64_t t = cand_offsets[b]; t < cand_offsets[b + 1]; ++t) owner[t] = b;
  parallel_for(total_C, threads, [&](int64_t t) {
    const int64_t b = owner[t];
    for (int32_t f = 0; f < F; ++f) {
      int64_t c = 0;
      if (b >= 0) {
        const int64_t us = b * F + f, is = t * F + f;
        for (int64_t i = user_offsets[us]; i < user_offsets[us + 1]; ++i)
          for (int64_t j = item_offsets[is]; j < item_offsets[is + 1]; ++j)
            c += (user_ids[i] == item_ids[j]) ? 1 : 0;
      }
      if (cap > 0 && c > cap) c = cap;
      counts[t * F + f] = static_cast<int32_t>(c);
    }
  });
}

// Independent second algorithm: multiplicity map of the user segment, summed over the
// item segment's ids.  Must agree exactly with oracle_hma_count.
void oracle_hma_count_hash(const int64_t* user_ids, const int64_t* user_offsets,
                           const int64_t* item_ids, const int64_t* item_offsets,
                           const int64_t* cand_offsets, int64_t B, int64_t total_C, int32_t F,
                           int32_t cap, int32_t* counts) {
  for (int64_t b = 0; b < B; ++b) {
    for (int32_t f = 0; f < F; ++f) {
      std::unordered_map<int64_t, int64_t> mult;
      const int64_t us = b * F + f;
      for (int64_t i = user_offsets[us]; i < user_offsets[us + 1]; ++i) mult[user_ids[i]] += 1;
      for (int64_t t = cand_offsets[b]; t < cand_offsets[b + 1]; ++t) {
        int64_t c = 0;
        const int64_t is = t * F + f;
        for (int64_t j = item_offsets[is]; j < item_offsets[is + 1]; ++j) {
          auto it = mult.find(item_ids[j]);
          if (it != mult.end()) c += it->second;
        }
        counts[t * F + f] = static_cast<int32_t>((cap > 0 && c > cap) ? cap : c);
      }
    }
  }
}

}  // extern "C"
