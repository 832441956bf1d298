// gsr/cuda_api.hpp — C++ host API over the B200 C-ABI (include/gsr_cuda.h).
//
// The reference's interface is in-process C++ (namespace gsr, typed
// exceptions: /root/reference/proj/include/gsr/common.hpp:13-35; SPEC op
// signatures SPEC.md:142-148,386-430,597-630). This header is the host-side
// mirror a reference caller (trainer.cpp / bench.cpp / verify.cpp,
// proj/CMakeLists.txt:23-25) links against: same names and error behaviour,
// every status code rethrown as the matching gsr:: exception. Header-only;
// link with -lgsrcuda (paper_2603_27156_b200/libgsrcuda.so).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../gsr_cuda.h"
#include "common.hpp"

namespace gsr {
namespace cuda {

enum class Mode : int { Alg12 = GSRC_MODE_ALG12, GsrC = GSRC_MODE_GSRC, Rev = GSRC_MODE_REV };
enum class Norm : int { None = GSRC_NORM_NONE, RowMean = GSRC_NORM_ROW_MEAN, SymDegree = GSRC_NORM_SYM_DEGREE };
enum class Precision : int { Fp32 = GSRC_GEMM_FP32, Tf32 = GSRC_GEMM_TF32 };

// RunConfig subset for the network.
struct NetConfig {
    Mode mode = Mode::GsrC;
    int layers = 8;
    int hidden = 64;
    int groups = 2;
    int k = 8;
    int d_in = 8;
    bool use_weight = true;
    bool use_bias = false;   // SPEC.md:289 (bias off by default)
    int index_source = 0;
    Precision precision = Precision::Fp32;
};

// optimizer_step config; Adam lr 1e-3 default.
struct OptimConfig {
    bool adam = true;
    float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, weight_decay = 0.f, momentum = 0.f;
};

// Maps a C-ABI status onto the reference's exception classes.
inline void check(int status, gsrc_ctx* ctx, const char* what) {
    if (status == GSRC_OK) return;
    std::string msg = std::string(what) + ": " + (ctx ? gsrc_last_error(ctx) : "no context");
    switch (status) {
        case GSRC_ERR_CONFIG: throw ConfigError(msg);
        case GSRC_ERR_SEQUENCING: throw SequencingError(msg);
        case GSRC_ERR_RESOURCE: throw ResourceError(msg);
        // an unexpected CUDA error is a device failure: the reference's
        // ResourceError class ("allocation / device", CLI exit 3)
        case GSRC_ERR_INTERNAL: throw ResourceError("internal CUDA error: " + msg);
        default: throw std::runtime_error(msg);
    }
}

// One device, one stream, one contiguous arena (SURVEY.md §8b Ownership).
class Context {
public:
    explicit Context(int device = 0) {
        const int st = gsrc_create(device, &h_);
        if (st != GSRC_OK) {
            if (st == GSRC_ERR_CONFIG) throw ConfigError("gsrc_create: bad device ordinal");
            throw ResourceError("gsrc_create: no usable CUDA device");
        }
    }
    ~Context() { gsrc_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    gsrc_ctx* handle() const { return h_; }

    // CsrGraph: int64 row_ptr, int32 col_idx ascending per row.
    void upload_graph(index_t n, const std::vector<index_t>& row_ptr, const std::vector<std::int32_t>& col_idx, Norm norm) {
        if (static_cast<index_t>(row_ptr.size()) != n + 1) throw ShapeError("row_ptr length != n + 1");
        check(gsrc_graph_upload(h_, n, static_cast<index_t>(col_idx.size()), row_ptr.data(), col_idx.data(), static_cast<int>(norm)), h_,
              "graph_upload");
    }
    void init_model(const NetConfig& c) {
        gsrc_model_cfg m{static_cast<int>(c.mode), c.layers, c.hidden, c.groups, c.k, c.d_in, c.use_weight, c.use_bias, c.index_source,
                         static_cast<int>(c.precision)};
        check(gsrc_model_init(h_, &m), h_, "model_init");
    }
    index_t num_params() const {
        int64_t n = 0;
        check(gsrc_num_params(h_, &n), h_, "num_params");
        return n;
    }
    void set_params(const std::vector<float>& p) { check(gsrc_params_set(h_, p.data(), static_cast<int64_t>(p.size())), h_, "params_set"); }
    std::vector<float> params() const {
        std::vector<float> p(static_cast<size_t>(num_params()));
        check(gsrc_params_get(h_, p.data(), static_cast<int64_t>(p.size())), h_, "params_get");
        return p;
    }
    std::vector<float> grads() const {
        std::vector<float> g(static_cast<size_t>(num_params()));
        check(gsrc_grads_get(h_, g.data(), static_cast<int64_t>(g.size())), h_, "grads_get");
        return g;
    }
    // NodeData: features n × d_in, labels n, train mask n.
    void upload_data(const float* x0, const float* y, const std::uint8_t* train_mask) {
        check(gsrc_data_upload(h_, x0, y, train_mask), h_, "data_upload");
    }
    void set_graph_capture(bool on) { check(gsrc_set_graph_capture(h_, on ? 1 : 0), h_, "set_graph_capture"); }

    // net_forward → ŷ.
    std::vector<float> forward(index_t n) {
        std::vector<float> yhat(static_cast<size_t>(n));
        check(gsrc_forward(h_, yhat.data()), h_, "forward");
        return yhat;
    }
    // net_forward + mse_loss + net_backward.
    double forward_backward() {
        double loss = 0;
        check(gsrc_forward_backward(h_, &loss), h_, "forward_backward");
        return loss;
    }
    void optimizer_step(const OptimConfig& o) {
        gsrc_optim_cfg c{o.adam ? 0 : 1, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, o.momentum};
        check(gsrc_optimizer_step(h_, &c), h_, "optimizer_step");
    }
    // cmd_train epoch body: forward → loss → backward → optimizer.
    double train_step(const OptimConfig& o) {
        gsrc_optim_cfg c{o.adam ? 0 : 1, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, o.momentum};
        double loss = 0;
        check(gsrc_train_step(h_, &c, &loss), h_, "train_step");
        return loss;
    }
    gsrc_timing last_timing() const {
        gsrc_timing t{};
        check(gsrc_last_timing(h_, &t), h_, "last_timing");
        return t;
    }
    // MemoryReport.
    gsrc_mem_report memory() const {
        gsrc_mem_report m{};
        check(gsrc_mem_stats(h_, &m), h_, "mem_stats");
        return m;
    }
    void high_water_reset() { check(gsrc_high_water_reset(h_), h_, "high_water_reset"); }

    // Optimizer state (Adam m, v, step) for exact resume beside a GSRP checkpoint.
    struct OptimState {
        std::vector<float> m, v;
        std::int64_t step = 0;
    };
    OptimState optim_state() const {
        OptimState o;
        const auto n = static_cast<size_t>(num_params());
        o.m.resize(n);
        o.v.resize(n);
        int64_t st = 0;
        check(gsrc_optim_state_get(h_, o.m.data(), o.v.data(), &st, static_cast<int64_t>(n)), h_, "optim_state_get");
        o.step = st;
        return o;
    }
    void set_optim_state(const OptimState& o) {
        if (o.m.size() != o.v.size()) throw ShapeError("optim state: m and v differ in length");
        check(gsrc_optim_state_set(h_, o.m.data(), o.v.data(), o.step, static_cast<int64_t>(o.m.size())), h_, "optim_state_set");
    }

    // Data parallelism: one process per GPU; rank 0 makes the
    // id, every rank joins with it; train_step then averages the gradients.
    static std::vector<unsigned char> comm_unique_id() {
        std::vector<unsigned char> id(128);
        check(gsrc_comm_unique_id(id.data(), id.size()), nullptr, "comm_unique_id");
        return id;
    }
    void comm_init(const std::vector<unsigned char>& id, int nranks, int rank) {
        check(gsrc_comm_init(h_, id.data(), nranks, rank), h_, "comm_init");
    }
    std::int64_t kernel_launches() const {
        int64_t n = 0;
        check(gsrc_kernel_launches(h_, &n), h_, "kernel_launches");
        return n;
    }
    // WorkCounter: {scalar_mul_adds, rows_touched} since create / work_reset()
    std::pair<std::uint64_t, std::uint64_t> work_counter() const {
        std::uint64_t ma = 0, rows = 0;
        check(gsrc_work_counter(h_, &ma, &rows), h_, "work_counter");
        return {ma, rows};
    }
    void work_reset() { check(gsrc_work_reset(h_), h_, "work_reset"); }

private:
    gsrc_ctx* h_ = nullptr;
};

}  // namespace cuda
}  // namespace gsr
