// schedule.cpp -- Lancet's weight-gradient computation schedule pass, at runtime (host C++).
//
// PAPER.md sec:dw_labelling / sec:dw_scheduling (L340-L398, Alg. 1):
//   * labelling: a dW instruction may overlap an all-to-all iff there is no directed path
//     between them in the dependency graph (L343) -- here by a breadth-first search from each
//     all-to-all over the graph and over its reverse;
//   * assignment: all-to-alls in program order; while the all-to-all's unoverlapped time
//     t_u > 0 and an unused eligible dW exists, take the dW minimising |t_u - t_W| (ties: the
//     lowest instruction index), t_u -= t_W (Alg. 1 lines 10-21);
//   * the caller then places each assigned dW right after its all-to-all's launch (L359).
// lancet_stack_dw_plan builds the backward program of an L-layer stack of this library's MoE
// layer (R17) and runs the pass on it, with per-op costs measured by the caller.
#include <cmath>
#include <cstdint>
#include <vector>

#include "lancet_moe.h"

#define LANCET_API extern "C" __attribute__((visibility("default")))

namespace {

enum { K_OTHER = 0, K_A2A = 1, K_DW = 2 };

// every node reachable from `src` along `adj` (src itself excluded unless on a cycle)
std::vector<char> bfs(const std::vector<std::vector<int>>& adj, int src)
{
    std::vector<char> seen(adj.size(), 0);
    std::vector<int> q(adj[src].begin(), adj[src].end());
    for (int v : q) seen[v] = 1;
    for (size_t h = 0; h < q.size(); ++h)
        for (int w : adj[q[h]])
            if (!seen[w]) { seen[w] = 1; q.push_back(w); }
    return seen;
}

int schedule(int n, const int32_t* kind, const double* cost, int n_edges, const int32_t* edges,
             int32_t* assign)
{
    std::vector<std::vector<int>> fwd(n), rev(n);
    for (int e = 0; e < n_edges; ++e) {
        const int s = edges[2 * e], t = edges[2 * e + 1];
        if (s < 0 || s >= n || t < 0 || t >= n) return 1;
        fwd[s].push_back(t);
        rev[t].push_back(s);
    }
    for (int i = 0; i < n; ++i) assign[i] = -1;
    std::vector<char> used(n, 0);
    for (int a = 0; a < n; ++a) {
        if (kind[a] != K_A2A) continue;
        const std::vector<char> desc = bfs(fwd, a), anc = bfs(rev, a);
        double t_u = cost[a];
        while (t_u > 0) {
            int best = -1;
            double bd = 0.0;
            for (int i = 0; i < n; ++i) {
                if (kind[i] != K_DW || used[i] || desc[i] || anc[i]) continue;
                const double dd = std::fabs(t_u - cost[i]);
                if (best < 0 || dd < bd) { best = i; bd = dd; }      // strict: ties -> lowest i
            }
            if (best < 0) break;
            t_u -= cost[best];
            used[best] = 1;
            assign[best] = a;
        }
    }
    return 0;
}

}  // namespace

LANCET_API lancet_status lancet_dw_schedule(int32_t n_instr, const int32_t* kind, const double* cost,
                                            int32_t n_edges, const int32_t* edges, int32_t* assign)
{
    if (n_instr < 0 || n_edges < 0 || (n_instr > 0 && (!kind || !cost || !assign)) || (n_edges > 0 && !edges))
        return LANCET_ERR_ARG;
    return schedule(n_instr, kind, cost, n_edges, edges, assign) ? LANCET_ERR_ARG : LANCET_OK;
}

LANCET_API lancet_status lancet_stack_dw_plan(int32_t L, int32_t n, const double* t_a2a, const double* t_dw,
                                              int32_t* host_layer, int32_t* host_a2a)
{
    if (L < 1 || n < 1 || !t_a2a || !t_dw || !host_layer || !host_a2a) return LANCET_ERR_ARG;
    // instruction ids, program order: layers L-1 .. 0, each K5[n] B1[n] DX[n] DW2 DW1 B2[n] K6 K7
    const int per = 4 * n + 4;
    auto id = [&](int l, int slot) { return (L - 1 - l) * per + slot; };
    auto K5 = [&](int l, int c) { return id(l, c); };
    auto B1 = [&](int l, int c) { return id(l, n + c); };
    auto DX = [&](int l, int c) { return id(l, 2 * n + c); };
    auto DW2 = [&](int l) { return id(l, 3 * n); };
    auto DW1 = [&](int l) { return id(l, 3 * n + 1); };
    auto B2 = [&](int l, int c) { return id(l, 3 * n + 2 + c); };
    auto K6 = [&](int l) { return id(l, 4 * n + 2); };
    auto K7 = [&](int l) { return id(l, 4 * n + 3); };
    const int N = L * per;
    std::vector<int32_t> kind(N, K_OTHER), edges;
    std::vector<double> cost(N, 0.0);
    auto edge = [&](int s, int t) { edges.push_back(s); edges.push_back(t); };
    for (int l = 0; l < L; ++l) {
        kind[DW2(l)] = kind[DW1(l)] = K_DW;
        cost[DW2(l)] = t_dw[2 * l];
        cost[DW1(l)] = t_dw[2 * l + 1];
        for (int c = 0; c < n; ++c) {
            kind[B1(l, c)] = kind[B2(l, c)] = K_A2A;
            cost[B1(l, c)] = t_a2a[(size_t)l * 2 * n + c];
            cost[B2(l, c)] = t_a2a[(size_t)l * 2 * n + n + c];
            edge(K5(l, c), B1(l, c));
            edge(B1(l, c), DX(l, c));
            edge(DX(l, c), B2(l, c));
            edge(B2(l, c), K6(l));
            edge(B1(l, c), DW2(l));     // dO received
            edge(B1(l, c), DW1(l));
            edge(DX(l, c), DW1(l));     // dA from the dX GEMMs
            edge(K5(l, c), K7(l));
            if (l > 0) edge(K6(l), K5(l - 1, c));   // dx of layer l = dy of layer l-1
        }
    }
    std::vector<int32_t> asg(N);
    if (schedule(N, kind.data(), cost.data(), (int)edges.size() / 2, edges.data(), asg.data()))
        return LANCET_ERR_ARG;
    for (int l = 0; l < L; ++l)
        for (int w = 0; w < 2; ++w) {
            const int a = asg[w == 0 ? DW2(l) : DW1(l)];
            host_layer[2 * l + w] = a < 0 ? -1 : L - 1 - a / per;
            host_a2a[2 * l + w] = a < 0 ? -1 : (a % per < 2 * n ? a % per - n : a % per - (3 * n + 2) + n);
        }
    return LANCET_OK;
}
