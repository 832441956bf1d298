// gsr/metrics.hpp — the four correlation metrics of the run report.
//
// SPEC.md:534-563 (module instrument): pearson, spearman (Pearson of
// average-tied ranks), kendall (tau-b, tie-corrected, O(m log m)) and r2
// (1 − SS_res/SS_tot, may be negative), reported per split on the
// test-mask nodes by default. Constant inputs give the explicit
// undefined marker NaN, never 0. Pure host functions in f64;
// the predictions come back from the device through gsrc_forward.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <vector>

#include "gsr/common.hpp"

namespace gsr {

struct CorrelationReport {
    double pearson = 0.0, spearman = 0.0, kendall = 0.0, r2 = 0.0;
    index_t count = 0;  // nodes the metrics ran over
};

namespace metrics_detail {
inline constexpr double undefined() { return std::numeric_limits<double>::quiet_NaN(); }

inline void check_pair(std::size_t na, std::size_t nb) {
    if (na != nb) throw ShapeError("metrics: vectors of different length");
    if (na < 2) throw ShapeError("metrics: need at least 2 values");
}

// average ranks (1-based) with ties sharing the mean of their positions
inline std::vector<double> average_ranks(const std::vector<double>& x) {
    const std::size_t n = x.size();
    std::vector<std::size_t> ord(n);
    std::iota(ord.begin(), ord.end(), std::size_t{0});
    std::stable_sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) { return x[a] < x[b]; });
    std::vector<double> r(n);
    for (std::size_t i = 0; i < n;) {
        std::size_t j = i + 1;
        while (j < n && x[ord[j]] == x[ord[i]]) ++j;
        const double avg = 0.5 * static_cast<double>(i + 1 + j);  // mean of positions i+1 .. j
        for (std::size_t q = i; q < j; ++q) r[ord[q]] = avg;
        i = j;
    }
    return r;
}

// pairs tied within runs of equal keys of a sorted sequence: Σ t(t−1)/2
template <class Eq>
inline std::int64_t tied_pairs(std::size_t n, Eq eq) {
    std::int64_t t = 0;
    for (std::size_t i = 0; i < n;) {
        std::size_t j = i + 1;
        while (j < n && eq(i, j)) ++j;
        const auto run = static_cast<std::int64_t>(j - i);
        t += run * (run - 1) / 2;
        i = j;
    }
    return t;
}

// inversions of v by merge sort (v is sorted on return)
inline std::int64_t count_inversions(std::vector<double>& v, std::vector<double>& tmp, std::size_t lo, std::size_t hi) {
    if (hi - lo < 2) return 0;
    const std::size_t mid = lo + (hi - lo) / 2;
    std::int64_t inv = count_inversions(v, tmp, lo, mid) + count_inversions(v, tmp, mid, hi);
    std::size_t i = lo, j = mid, o = lo;
    while (i < mid && j < hi) {
        if (v[j] < v[i]) {
            inv += static_cast<std::int64_t>(mid - i);
            tmp[o++] = v[j++];
        } else {
            tmp[o++] = v[i++];
        }
    }
    while (i < mid) tmp[o++] = v[i++];
    while (j < hi) tmp[o++] = v[j++];
    std::copy(tmp.begin() + static_cast<std::ptrdiff_t>(lo), tmp.begin() + static_cast<std::ptrdiff_t>(hi), v.begin() + static_cast<std::ptrdiff_t>(lo));
    return inv;
}
}  // namespace metrics_detail

// sample Pearson correlation
inline double pearson(const std::vector<double>& a, const std::vector<double>& b) {
    metrics_detail::check_pair(a.size(), b.size());
    const double n = static_cast<double>(a.size());
    double ma = 0.0, mb = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) { ma += a[i]; mb += b[i]; }
    ma /= n;
    mb /= n;
    double sab = 0.0, saa = 0.0, sbb = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double da = a[i] - ma, db = b[i] - mb;
        sab += da * db;
        saa += da * da;
        sbb += db * db;
    }
    if (saa == 0.0 || sbb == 0.0) return metrics_detail::undefined();
    return std::max(-1.0, std::min(1.0, sab / std::sqrt(saa * sbb)));
}

// Pearson of average-tied ranks
inline double spearman(const std::vector<double>& a, const std::vector<double>& b) {
    metrics_detail::check_pair(a.size(), b.size());
    return pearson(metrics_detail::average_ranks(a), metrics_detail::average_ranks(b));
}

// Kendall tau-b in O(m log m) (Knight's algorithm):
// tau_b = (n0 − n1 − n2 + n3 − 2·swaps) / sqrt((n0 − n1)(n0 − n2)), with n1 / n2
// the pairs tied in a / b, n3 the pairs tied in both, swaps the discordant
// pairs counted as inversions of b after sorting by (a, b).
inline double kendall(const std::vector<double>& a, const std::vector<double>& b) {
    metrics_detail::check_pair(a.size(), b.size());
    const std::size_t n = a.size();
    std::vector<std::size_t> ord(n);
    std::iota(ord.begin(), ord.end(), std::size_t{0});
    std::sort(ord.begin(), ord.end(), [&](std::size_t x, std::size_t y) { return a[x] < a[y] || (a[x] == a[y] && b[x] < b[y]); });
    std::vector<double> sa(n), sb(n);
    for (std::size_t i = 0; i < n; ++i) { sa[i] = a[ord[i]]; sb[i] = b[ord[i]]; }
    const std::int64_t n0 = static_cast<std::int64_t>(n) * static_cast<std::int64_t>(n - 1) / 2;
    const std::int64_t n1 = metrics_detail::tied_pairs(n, [&](std::size_t i, std::size_t j) { return sa[i] == sa[j]; });
    const std::int64_t n3 = metrics_detail::tied_pairs(n, [&](std::size_t i, std::size_t j) { return sa[i] == sa[j] && sb[i] == sb[j]; });
    std::vector<double> tmp(n);
    const std::int64_t swaps = metrics_detail::count_inversions(sb, tmp, 0, n);  // sb is sorted afterwards
    const std::int64_t n2 = metrics_detail::tied_pairs(n, [&](std::size_t i, std::size_t j) { return sb[i] == sb[j]; });
    const double den = std::sqrt(static_cast<double>(n0 - n1) * static_cast<double>(n0 - n2));  // sqrt(x·x) == x exactly
    if (den == 0.0) return metrics_detail::undefined();
    const double num = static_cast<double>(n0 - n1 - n2 + n3) - 2.0 * static_cast<double>(swaps);
    return std::max(-1.0, std::min(1.0, num / den));
}

// coefficient of determination 1 − SS_res/SS_tot
inline double r2(const std::vector<double>& pred, const std::vector<double>& truth) {
    metrics_detail::check_pair(pred.size(), truth.size());
    double m = 0.0;
    for (double t : truth) m += t;
    m /= static_cast<double>(truth.size());
    double ss_res = 0.0, ss_tot = 0.0;
    for (std::size_t i = 0; i < truth.size(); ++i) {
        ss_res += (truth[i] - pred[i]) * (truth[i] - pred[i]);
        ss_tot += (truth[i] - m) * (truth[i] - m);
    }
    if (ss_tot == 0.0) return metrics_detail::undefined();
    return 1.0 - ss_res / ss_tot;
}

// The report over the nodes whose mask byte equals `split` (default: every
// node with a nonzero mask byte when split < 0).
inline CorrelationReport correlate(const float* pred, const float* truth, const std::uint8_t* mask, index_t n, int split = -1) {
    std::vector<double> p, t;
    for (index_t i = 0; i < n; ++i) {
        const bool take = mask == nullptr || (split < 0 ? mask[i] != 0 : mask[i] == split);
        if (!take) continue;
        p.push_back(pred[i]);
        t.push_back(truth[i]);
    }
    CorrelationReport r;
    r.count = static_cast<index_t>(p.size());
    if (p.size() < 2) {
        r.pearson = r.spearman = r.kendall = r.r2 = metrics_detail::undefined();
        return r;
    }
    r.pearson = pearson(p, t);
    r.spearman = spearman(p, t);
    r.kendall = kendall(p, t);
    r.r2 = r2(p, t);
    return r;
}

}  // namespace gsr
