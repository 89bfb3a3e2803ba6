// softmax_pin.cpp — TEST INFRASTRUCTURE: pins the float oracle's per-token
// log-softmax quantities (A1: logp, ref_logp, entropy, KL) to the
// reference's OWN fp64 softmax, yatt::distattn::reference_attention
// (proj/src/distattn.cpp:79-123: max-subtracted row softmax in fp64, then
// the probability-weighted sum of V).  The reference has no log-prob code,
// but its attention oracle is exactly "softmax over a row of scores, then an
// expectation", so one head per token row gives every quantity A1 needs:
//
//   head_dim 4 (scale 1/sqrt(4) = 0.5, exact), q_i = (2, 0, 0, 0) for every
//   query i, k_j = (x_j, 0, 0, 0) -> score_ij = x_j exactly;
//   v_j = (x_j, [j == y], z_j, 1)  ->  output row 0 =
//         (E_p[x], p_y, E_p[z], 1)    with p = softmax(x)
//
// and the same head with x <-> z for the reference logits.  Derived values
// (tests/test_oracle_float.py): logp = ln p_y, lse_p = x_y - logp,
// H = lse_p - E_p[x], full KL(p || q) = E_p[x] - lse_p - E_p[z] + lse_q.
//
// stdin (binary, little-endian): int32 rows, int32 V, rows*V float64 policy
// logits, rows*V float64 reference logits, rows int32 targets.
// stdout: one line per (row, tensor): "row tensor c0 c1 c2 c3" (%.17g).
// Linked against oracle/_ref/libyatt_ref.a (oracle/Makefile softmax_pin).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "yatt/distattn.hpp"

using namespace yatt::distattn;

// `softmax_pin lmhead`: the fused LM-head path (§8f #4) the same way — one
// head per token row with q_i = sqrt(d) h (d a power of 4: exact scale),
// k_j = W_j (the vocabulary rows), so score_j = h . W_j: head A with
// v_j = W_j gives E_p[W] (E_p[logit] = h . E_p[W]); head B with
// v_j = ([j == y], 0, ...) gives p_y.
// stdin: int32 rows, d, V; rows*d float64 hidden; V*d float64 W; rows int32
// targets.  stdout per row: "row p_y E_p[W]_0 ... E_p[W]_{d-1}".
static int lmhead_main() {
  int32_t rows = 0, d = 0, V = 0;
  if (std::fread(&rows, 4, 1, stdin) != 1 || std::fread(&d, 4, 1, stdin) != 1 ||
      std::fread(&V, 4, 1, stdin) != 1 || rows <= 0 || d <= 0 || V <= 0)
    return 2;
  std::vector<double> h(size_t(rows) * d), w(size_t(V) * d);
  std::vector<int32_t> tgt(static_cast<size_t>(rows));
  if (std::fread(h.data(), 8, h.size(), stdin) != h.size() ||
      std::fread(w.data(), 8, w.size(), stdin) != w.size() ||
      std::fread(tgt.data(), 4, tgt.size(), stdin) != tgt.size())
    return 2;
  const double sq = std::sqrt(double(d));
  for (int32_t r = 0; r < rows; ++r) {
    double py = 0;
    std::vector<double> ew(static_cast<size_t>(d));
    for (int head = 0; head < 2; ++head) {
      AttentionProblem pb;
      pb.seq_len = V;
      pb.head_dim = d;
      pb.num_heads = 1;
      pb.q = Tensor3(1, V, d);
      pb.k = Tensor3(1, V, d);
      pb.v = Tensor3(1, V, d);
      for (int j = 0; j < V; ++j)
        for (int c = 0; c < d; ++c) {
          pb.q.at(0, j, c) = sq * h[size_t(r) * d + c];
          pb.k.at(0, j, c) = w[size_t(j) * d + c];
          pb.v.at(0, j, c) = head == 0 ? w[size_t(j) * d + c]
                                       : (c == 0 && j == tgt[size_t(r)] ? 1.0 : 0.0);
        }
      const Tensor3 o = reference_attention(pb);
      if (head == 0)
        for (int c = 0; c < d; ++c) ew[size_t(c)] = o.at(0, 0, c);
      else
        py = o.at(0, 0, 0);
    }
    std::printf("%d %.17g", r, py);
    for (int c = 0; c < d; ++c) std::printf(" %.17g", ew[size_t(c)]);
    std::printf("\n");
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "lmhead") return lmhead_main();
  int32_t rows = 0, V = 0;
  if (std::fread(&rows, 4, 1, stdin) != 1 || std::fread(&V, 4, 1, stdin) != 1 || rows <= 0 ||
      V <= 0)
    return 2;
  const size_t n = size_t(rows) * size_t(V);
  std::vector<double> pol(n), ref(n);
  std::vector<int32_t> tgt(static_cast<size_t>(rows));
  if (std::fread(pol.data(), 8, n, stdin) != n || std::fread(ref.data(), 8, n, stdin) != n ||
      std::fread(tgt.data(), 4, size_t(rows), stdin) != size_t(rows))
    return 2;
  for (int32_t r = 0; r < rows; ++r) {
    for (int t = 0; t < 2; ++t) {
      const double* x = (t == 0 ? pol.data() : ref.data()) + size_t(r) * V;  // scores
      const double* z = (t == 0 ? ref.data() : pol.data()) + size_t(r) * V;  // the other tensor
      AttentionProblem pb;
      pb.seq_len = V;
      pb.head_dim = 4;
      pb.num_heads = 1;
      pb.q = Tensor3(1, V, 4);
      pb.k = Tensor3(1, V, 4);
      pb.v = Tensor3(1, V, 4);
      for (int j = 0; j < V; ++j) {
        pb.q.at(0, j, 0) = 2.0;
        pb.k.at(0, j, 0) = x[j];
        pb.v.at(0, j, 0) = x[j];
        pb.v.at(0, j, 1) = j == tgt[size_t(r)] ? 1.0 : 0.0;
        pb.v.at(0, j, 2) = z[j];
        pb.v.at(0, j, 3) = 1.0;
      }
      const Tensor3 o = reference_attention(pb);
      std::printf("%d %d %.17g %.17g %.17g %.17g\n", r, t, o.at(0, 0, 0), o.at(0, 0, 1),
                  o.at(0, 0, 2), o.at(0, 0, 3));
    }
  }
  return 0;
}
