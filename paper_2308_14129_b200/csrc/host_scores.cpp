// Link-prediction metrics over the scores of every partition (SURVEY §8e(3),
// §8f #2): evaluation routes each val/test edge to every partition holding
// both endpoints (assign_eval_edges, partitioner.cpp:212-242), each partition
// scores its edges on its own GPU (spd_tgn_evaluate), and the caller gathers
// the (positive, negative) score lists of all ranks; the global AP and AUC
// are then one pass over the merged, sorted scores.
//
// Definitions (those of the TIG literature's evaluation, sklearn's
// average_precision_score / roc_auc_score): scores sorted descending and
// grouped by equal value; AP = sum over groups of (R_g - R_{g-1}) * P_g with
// precision / recall at each group's end; AUC = trapezoidal area under the
// ROC curve over the same groups (ties count one half), / (n_pos * n_neg).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "capi_types.hpp"
#include "host.hpp"

using namespace spd;

extern "C" spd_status spd_link_metrics(const float* pos, uint64_t n_pos, const float* neg, uint64_t n_neg,
                                       double* ap, double* auc) {
    GUARD({
        if (n_pos == 0 || n_neg == 0) data_error("InvalidParams", "link metrics need positive and negative scores");
        if ((!pos || !neg) || (!ap && !auc)) usage_error("null score or output pointer");
        struct Item {
            float s;
            std::uint8_t y;
        };
        std::vector<Item> v;
        v.reserve(n_pos + n_neg);
        for (uint64_t i = 0; i < n_pos; ++i) v.push_back({pos[i], 1});
        for (uint64_t i = 0; i < n_neg; ++i) v.push_back({neg[i], 0});
        for (const Item& it : v)
            if (std::isnan(it.s)) data_error("InvalidParams", "NaN score");
        std::sort(v.begin(), v.end(), [](const Item& a, const Item& b) { return a.s > b.s; });
        double tp = 0, fp = 0, a_ap = 0, a_auc = 0, prev_r = 0, prev_tp = 0, prev_fp = 0;
        const double P = double(n_pos), N = double(n_neg);
        for (std::size_t i = 0; i < v.size();) {
            std::size_t j = i;
            while (j < v.size() && v[j].s == v[i].s) {
                (v[j].y ? tp : fp) += 1.0;
                ++j;
            }
            const double r = tp / P;
            a_ap += (r - prev_r) * (tp / (tp + fp));
            a_auc += (fp - prev_fp) * (tp + prev_tp) * 0.5;
            prev_r = r;
            prev_tp = tp;
            prev_fp = fp;
            i = j;
        }
        if (ap) *ap = a_ap;
        if (auc) *auc = a_auc / (P * N);
    });
}
