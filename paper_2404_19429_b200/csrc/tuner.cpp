// tuner.cpp -- the chunk-count search of Lancet's operator partition pass at the scope of one
// MoE layer, host only.
//
//   * T(n) = min over partition counts: the layer is one partition range, so the
//     DP over ranges reduces to a scan over n = 1..K (K = the maximum number of partitions).
//   * P(i, n, k) comes from the pipeline scheduler: the stages of every chunk are
//     placed on a computation and a communication lane in their scheduled order; an op starts
//     at the later of (i) the end of the ops it depends on and (ii) the end of the previous op
//     of its lane; the step time is the end of the last op.
//   * Op costs come from a caching profiler ("profiling is done once for each
//     (partitioned) operation with the same shape"): per-op durations measured at a few
//     profiled chunk counts.  Communication uses the paper's cost model: costs
//     at several message sizes, linearly interpolated, and an n-partitioned all-to-all of
//     capacity C costs the model at C/n.  Computation at an unprofiled n is interpolated
//     linearly in 1/n (per-chunk cost = fixed + whole / n between profiled points).
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/lancet_moe.h"

namespace {

struct Pt {
    double x, y;
};

// piecewise-linear interpolation through points sorted by x; linear extrapolation with the end
// segments; never negative
double interp(std::vector<Pt> p, double x)
{
    std::sort(p.begin(), p.end(), [](const Pt& a, const Pt& b) { return a.x < b.x; });
    if (p.size() == 1) return std::max(0.0, p[0].x > 0 ? p[0].y * x / p[0].x : p[0].y);
    size_t i = 1;
    while (i + 1 < p.size() && x > p[i].x) ++i;
    const Pt& a = p[i - 1];
    const Pt& b = p[i];
    const double t = b.x != a.x ? (x - a.x) / (b.x - a.x) : 0.0;
    return std::max(0.0, a.y + t * (b.y - a.y));
}

bool is_comm(int op)
{
    return op == LANCET_OP_COUNTS || op == LANCET_OP_DISPATCH || op == LANCET_OP_COMBINE ||
           op == LANCET_OP_BWD_DISPATCH || op == LANCET_OP_BWD_COMBINE;
}
bool once(int op) { return op == LANCET_OP_GATE || op == LANCET_OP_COUNTS || op == LANCET_OP_K7; }

struct Sim {
    double lane[2] = {0.0, 0.0};                       // 0 computation, 1 communication
    std::vector<std::pair<double, double>> busy[2];    // by op kind (exposure)
    double run(int lane_id, int kind, double cost, std::initializer_list<double> deps, double after = 0.0)
    {
        double s = std::max(lane[lane_id], after);
        for (double d : deps) s = std::max(s, d);
        const double e = s + cost;
        lane[lane_id] = e;
        busy[kind].push_back({s, e});
        return e;
    }
};

double union_len(std::vector<std::pair<double, double>> v, std::vector<std::pair<double, double>>* out = nullptr)
{
    std::sort(v.begin(), v.end());
    std::vector<std::pair<double, double>> u;
    for (auto& iv : v) {
        if (!u.empty() && iv.first <= u.back().second) u.back().second = std::max(u.back().second, iv.second);
        else u.push_back(iv);
    }
    double t = 0.0;
    for (auto& iv : u) t += iv.second - iv.first;
    if (out) *out = u;
    return t;
}

// one fwd + bwd of the layer with n chunks on the schedule of lancet.cu; cost(op) per chunk
// (per step for once-ops); returns the step time and the exposed communication
template <typename Cost>
void simulate(int schedule, int n, Cost cost, double* step, double* exposed)
{
    Sim s;
    const int C = 0, M = 1;
    std::vector<double> disp(n), fc2(n), comb(n), b1(n), dfc1(n), b2(n);
    const double g = s.run(C, C, cost(LANCET_OP_GATE), {});
    const double cnt = s.run(M, M, cost(LANCET_OP_COUNTS), {g});
    if (schedule == 0) {
        // per-chunk launches, host-planned (pull / NCCL): the host waits for the counts; stage
        // order D0..Dn-1, C0..Cn-1; dW of chunk c right after its dX
        for (int c = 0; c < n; ++c) disp[c] = s.run(M, M, cost(LANCET_OP_DISPATCH), {cnt});
        for (int c = 0; c < n; ++c) {
            const double a = s.run(C, C, cost(LANCET_OP_FC1), {disp[c]}, cnt);
            fc2[c] = s.run(C, C, cost(LANCET_OP_FC2), {a});
        }
        for (int c = 0; c < n; ++c) comb[c] = s.run(M, M, cost(LANCET_OP_COMBINE), {fc2[c]});
        for (int c = 0; c < n; ++c) s.run(C, C, cost(LANCET_OP_GATHER), {comb[c]});
        std::vector<double> k5(n);
        for (int c = 0; c < n; ++c) k5[c] = s.run(C, C, cost(LANCET_OP_K5), {});
        for (int c = 0; c < n; ++c) b1[c] = s.run(M, M, cost(LANCET_OP_BWD_DISPATCH), {k5[c]});
        for (int c = 0; c < n; ++c) {
            const double a = s.run(C, C, cost(LANCET_OP_DFC2), {b1[c]});
            dfc1[c] = s.run(C, C, cost(LANCET_OP_DFC1), {a});
            s.run(C, C, cost(LANCET_OP_DW), {dfc1[c]});
        }
        for (int c = 0; c < n; ++c) b2[c] = s.run(M, M, cost(LANCET_OP_BWD_COMBINE), {dfc1[c]});
        for (int c = 0; c < n; ++c) s.run(C, C, cost(LANCET_OP_K6), {b2[c]});
        s.run(C, C, cost(LANCET_OP_K7), {});
    } else {
        // push pipeline: the fused exchange kernels on the comm stream; fc1 / dfc2 one launch
        // over all chunks (waiting per chunk on the device), fc2 / dfc1 per chunk; dW merged
        for (int c = 0; c < n; ++c) disp[c] = s.run(M, M, cost(LANCET_OP_DISPATCH), {cnt});
        double f1 = 0.0;
        for (int c = 0; c < n; ++c) f1 = s.run(C, C, cost(LANCET_OP_FC1), {disp[c], cnt});
        for (int c = 0; c < n; ++c) fc2[c] = s.run(C, C, cost(LANCET_OP_FC2), {f1});
        double lastc = 0.0;
        for (int c = 0; c < n; ++c) lastc = comb[c] = s.run(M, M, cost(LANCET_OP_COMBINE), {fc2[c]});
        for (int c = 0; c < n; ++c) b1[c] = s.run(M, M, cost(LANCET_OP_BWD_DISPATCH), {lastc});
        s.run(M, C, cost(LANCET_OP_K7), {b1[n - 1]});             // K7 beside the dX GEMMs
        double d2 = 0.0;
        for (int c = 0; c < n; ++c) d2 = s.run(C, C, cost(LANCET_OP_DFC2), {b1[c]});
        for (int c = 0; c < n; ++c) dfc1[c] = s.run(C, C, cost(LANCET_OP_DFC1), {d2});
        s.run(C, C, cost(LANCET_OP_DW), {dfc1[n - 1]});
        for (int c = 0; c < n; ++c) s.run(M, M, cost(LANCET_OP_BWD_COMBINE), {dfc1[c]});
    }
    *step = std::max(s.lane[0], s.lane[1]);
    std::vector<std::pair<double, double>> comm, comp;
    const double tc = union_len(s.busy[1], &comm);
    union_len(s.busy[0], &comp);
    double cover = 0.0;
    for (auto& a : comm)
        for (auto& b : comp) cover += std::max(0.0, std::min(a.second, b.second) - std::max(a.first, b.first));
    *exposed = tc - cover;
}

}  // namespace

extern "C" __attribute__((visibility("default"))) lancet_status
lancet_tune_chunks(const lancet_tune_input* in, double* pred_us, double* pred_exposed_us, int32_t* best_n)
{
    if (!in || !pred_us || !best_n || in->n_prof < 2 || !in->prof_n || !in->prof_us || in->max_chunks < 1 ||
        in->max_chunks > 64 || !(in->bytes_full > 0.0) || (in->schedule != 0 && in->schedule != 1))
        return LANCET_ERR_ARG;
    for (int i = 0; i < in->n_prof; ++i)
        if (in->prof_n[i] < 1) return LANCET_ERR_ARG;
    double best = 0.0;
    *best_n = 0;
    for (int n = 1; n <= in->max_chunks; ++n) {
        auto cost = [&](int op) -> double {
            std::vector<Pt> pts;
            for (int i = 0; i < in->n_prof; ++i) {
                const double y = in->prof_us[(size_t)i * LANCET_OP_N + op];
                if (once(op)) pts.push_back({(double)in->prof_n[i], y});
                else if (is_comm(op)) pts.push_back({in->bytes_full / in->prof_n[i], y});   // size model
                else pts.push_back({1.0 / in->prof_n[i], y});                              // fixed + whole/n
            }
            if (once(op)) {                     // once per step: the mean of the profiles
                double m = 0.0;
                for (auto& p : pts) m += p.y;
                return m / pts.size();
            }
            if (op == LANCET_OP_DW && in->schedule == 1) return interp(pts, 1.0 / n) * n;   // merged: whole
            return is_comm(op) ? interp(pts, in->bytes_full / n) : interp(pts, 1.0 / n);
        };
        double st, ex;
        simulate(in->schedule, n, cost, &st, &ex);
        pred_us[n - 1] = st;
        if (pred_exposed_us) pred_exposed_us[n - 1] = ex;
        if (*best_n == 0 || st < best) { best = st; *best_n = n; }
    }
    return LANCET_OK;
}
