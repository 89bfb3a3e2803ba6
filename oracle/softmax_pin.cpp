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
#include <cstdint>
#include <cstdio>
#include <vector>

#include "yatt/distattn.hpp"

using namespace yatt::distattn;

int main() {
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
