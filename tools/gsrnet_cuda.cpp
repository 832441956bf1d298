// gsrnet-cuda — C++ host CLI for the B200 GSR-GNN training step.
//
// Mirrors the reference's `gsrnet train` (cmd_train SPEC.md:597-605; flags
// SPEC.md:645; exit codes 0/1/3 SPEC.md:647) for the one path this build
// accelerates: it reads a graph-store GSRG graph and GSRN node file
// (SPEC.md:215-218), configures the network, and runs full-batch epochs
// (forward → masked MSE → backward with inverse recomputation → Adam) through
// the C++ host API (include/gsr/cuda_api.hpp) over the C-ABI. One line-delimited
// JSON record per epoch plus a summary record (RunReport SPEC.md:591-594).
//
//   gsrnet-cuda train --graph g.gsrg --nodes n.gsrn [--model gsrc|gsr|baseline]
//       [--layers L] [--hidden D] [--groups C] [--k K] [--epochs E] [--lr LR]
//       [--norm none|row_mean|sym] [--precision fp32|tf32] [--seed S]
//       [--params init.f32 | --resume in.gsrp] [--checkpoint out.gsrp]
//       [--report out.jsonl] [--device I] [--threads T]
//       [--nranks N --rank R --comm-file F]
//
// After the last epoch a "metrics" record carries the CorrelationReport
// (Pearson, Spearman, Kendall tau-b, R²) of the predictions
// per split (train / val / test; test is the SPEC default). --checkpoint also
// writes the Adam state (m, v, step) to <out>.adam so --resume continues the
// interrupted trajectory exactly (GSRP itself holds parameters only,
// SPEC.md:293). Data parallelism: one process per GPU, each with its own graph
// and node files; rank 0 writes the NCCL id to --comm-file, the others read it,
// and every step averages the gradients over the ranks.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gsr/cuda_api.hpp"
#include "gsr/metrics.hpp"
#include "gsr/threads.hpp"

namespace {

using gsr::index_t;

std::vector<char> slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw gsr::ResourceError("cannot open " + path);
    return std::vector<char>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

template <typename T>
T get_le(const std::vector<char>& b, size_t off) {  // x86-64 / aarch64 hosts are little-endian
    T v;
    std::memcpy(&v, b.data() + off, sizeof(T));
    return v;
}

struct Graph {
    index_t n = 0;
    std::vector<index_t> row_ptr;
    std::vector<std::int32_t> col_idx;
};

// GSRG: "GSRG", u32 version, u64 n, u64 e, row_ptr i64[n+1], col_idx i32[e].
Graph read_gsrg(const std::string& path) {
    const auto b = slurp(path);
    if (b.size() < 24 || std::memcmp(b.data(), "GSRG", 4) != 0) throw gsr::FormatError(path + ": bad GSRG magic");
    if (get_le<std::uint32_t>(b, 4) != 1) throw gsr::FormatError(path + ": unsupported GSRG version");
    Graph g;
    g.n = static_cast<index_t>(get_le<std::uint64_t>(b, 8));
    const auto e = static_cast<index_t>(get_le<std::uint64_t>(b, 16));
    const size_t need = 24 + 8 * static_cast<size_t>(g.n + 1) + 4 * static_cast<size_t>(e);
    if (b.size() != need) throw gsr::FormatError(path + ": truncated GSRG");
    g.row_ptr.resize(static_cast<size_t>(g.n + 1));
    g.col_idx.resize(static_cast<size_t>(e));
    std::memcpy(g.row_ptr.data(), b.data() + 24, 8 * g.row_ptr.size());
    std::memcpy(g.col_idx.data(), b.data() + 24 + 8 * g.row_ptr.size(), 4 * g.col_idx.size());
    return g;
}

struct Nodes {
    index_t n = 0, d_in = 0;
    std::vector<float> x, y;
    std::vector<std::uint8_t> train, split;
    index_t split_count[3] = {0, 0, 0};
};

// GSRN: "GSRN", u64 n, u64 d_in, f64 features, f64 labels, u8 split.
Nodes read_gsrn(const std::string& path, gsr::ThreadPool* pool) {
    const auto b = slurp(path);
    if (b.size() < 20 || std::memcmp(b.data(), "GSRN", 4) != 0) throw gsr::FormatError(path + ": bad GSRN magic");
    Nodes d;
    d.n = static_cast<index_t>(get_le<std::uint64_t>(b, 4));
    d.d_in = static_cast<index_t>(get_le<std::uint64_t>(b, 12));
    const size_t n = static_cast<size_t>(d.n), di = static_cast<size_t>(d.d_in);
    if (b.size() != 20 + 8 * n * di + 8 * n + n) throw gsr::FormatError(path + ": truncated GSRN");
    d.x.resize(n * di);
    d.y.resize(n);
    d.train.resize(n);
    d.split.resize(n);
    // f64 → f32 decode, row-partitioned over the host pool
    gsr::parallel_for(pool, d.n, [&](index_t lo, index_t hi) {
        for (size_t i = static_cast<size_t>(lo); i < static_cast<size_t>(hi); ++i) {
            for (size_t j = 0; j < di; ++j) d.x[i * di + j] = static_cast<float>(get_le<double>(b, 20 + 8 * (i * di + j)));
            d.y[i] = static_cast<float>(get_le<double>(b, 20 + 8 * n * di + 8 * i));
            d.split[i] = static_cast<std::uint8_t>(b[20 + 8 * n * di + 8 * n + i]);
        }
    });
    for (size_t i = 0; i < n; ++i) {
        const auto s = d.split[i];
        if (s > 2) throw gsr::FormatError(path + ": split code out of range");
        d.train[i] = s == 0;
        d.split_count[s]++;
    }
    return d;
}

// Seeded init, same scales as paper_2603_27156_b200/model.py init_params
// (Glorot encoder/head, blocks ±sqrt(6/2w)/sqrt(L·C)); splitmix64 stream.
std::vector<float> init_params(const gsr::cuda::NetConfig& c, index_t P, std::uint64_t seed) {
    std::uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
    auto uni = [&](double lim) {
        s += 0x9E3779B97F4A7C15ull;
        std::uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        return static_cast<float>((static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0) * lim);
    };
    const int C = c.mode == gsr::cuda::Mode::Alg12 ? 2 : c.groups;
    const int D = c.hidden, w = D / C;
    std::vector<float> p(static_cast<size_t>(P), 0.f);
    size_t o = 0;
    const double se = std::sqrt(6.0 / (c.d_in + D));
    for (int i = 0; i < c.d_in * D; ++i) p[o++] = uni(se);
    o += static_cast<size_t>(D);
    const double bs = std::sqrt(6.0 / (2.0 * w)) / std::sqrt(static_cast<double>(std::max(1, c.layers * C)));
    for (int l = 0; l < c.layers; ++l)
        for (int i = 0; i < C; ++i) {
            for (int j = 0; j < w * w; ++j) p[o++] = uni(bs);
            o += static_cast<size_t>(w);
        }
    const double sh = std::sqrt(6.0 / (D + 1));
    for (int i = 0; i < D; ++i) p[o++] = uni(sh);
    return p;
}

// GSRP checkpoint, same layout as paper_2603_27156_b200/model.py:
// "GSRP", u32 version 1, u64 mode, L, D, C, d_in, block count; per block u64 rows,
// cols, then w (rows × cols) and b (cols) as f64. Blocks: encoder, layer blocks, head.
struct BlockSpan { size_t off, rows, cols; };
std::vector<BlockSpan> gsrp_blocks(const gsr::cuda::NetConfig& c) {
    const int C = c.mode == gsr::cuda::Mode::Alg12 ? 2 : c.groups;
    const size_t D = static_cast<size_t>(c.hidden), w = D / static_cast<size_t>(C), din = static_cast<size_t>(c.d_in);
    std::vector<BlockSpan> b;
    size_t o = 0;
    b.push_back({o, din, D});
    o += din * D + D;
    for (int l = 0; l < c.layers; ++l)
        for (int i = 0; i < C; ++i) { b.push_back({o, w, w}); o += w * w + w; }
    b.push_back({o, D, 1});
    return b;
}

void write_gsrp(const std::string& path, const std::vector<float>& p, const gsr::cuda::NetConfig& c) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw gsr::ResourceError("cannot write " + path);
    const auto blocks = gsrp_blocks(c);
    auto u64 = [&](std::uint64_t v) { f.write(reinterpret_cast<const char*>(&v), 8); };
    f.write("GSRP", 4);
    const std::uint32_t ver = 1;
    f.write(reinterpret_cast<const char*>(&ver), 4);
    u64(static_cast<std::uint64_t>(c.mode)); u64(static_cast<std::uint64_t>(c.layers)); u64(static_cast<std::uint64_t>(c.hidden));
    u64(static_cast<std::uint64_t>(c.mode == gsr::cuda::Mode::Alg12 ? 2 : c.groups)); u64(static_cast<std::uint64_t>(c.d_in)); u64(blocks.size());
    for (const auto& b : blocks) {
        u64(b.rows); u64(b.cols);
        for (size_t i = 0; i < b.rows * b.cols + b.cols; ++i) {
            const double v = p[b.off + i];
            f.write(reinterpret_cast<const char*>(&v), 8);
        }
    }
}

std::vector<float> read_gsrp(const std::string& path, const gsr::cuda::NetConfig& c, index_t P) {
    const auto buf = slurp(path);
    if (buf.size() < 56 || std::memcmp(buf.data(), "GSRP", 4) != 0) throw gsr::FormatError(path + ": bad GSRP magic");
    if (get_le<std::uint32_t>(buf, 4) != 1) throw gsr::FormatError(path + ": unsupported GSRP version");
    const std::uint64_t want[5] = {static_cast<std::uint64_t>(c.mode), static_cast<std::uint64_t>(c.layers), static_cast<std::uint64_t>(c.hidden),
                                   static_cast<std::uint64_t>(c.mode == gsr::cuda::Mode::Alg12 ? 2 : c.groups), static_cast<std::uint64_t>(c.d_in)};
    for (int i = 0; i < 5; ++i)
        if (get_le<std::uint64_t>(buf, 8 + 8 * i) != want[i]) throw gsr::ShapeError(path + ": checkpoint config differs from the run config");
    const auto blocks = gsrp_blocks(c);
    if (get_le<std::uint64_t>(buf, 48) != blocks.size()) throw gsr::FormatError(path + ": block count mismatch");
    std::vector<float> p(static_cast<size_t>(P), 0.f);
    size_t off = 56;
    for (const auto& b : blocks) {
        if (off + 16 > buf.size() || get_le<std::uint64_t>(buf, off) != b.rows || get_le<std::uint64_t>(buf, off + 8) != b.cols)
            throw gsr::FormatError(path + ": block shape mismatch or truncation");
        off += 16;
        const size_t cnt = b.rows * b.cols + b.cols;
        if (off + 8 * cnt > buf.size()) throw gsr::FormatError(path + ": truncated GSRP");
        for (size_t i = 0; i < cnt; ++i) p[b.off + i] = static_cast<float>(get_le<double>(buf, off + 8 * i));
        off += 8 * cnt;
    }
    if (off != buf.size()) throw gsr::FormatError(path + ": trailing bytes in GSRP");
    return p;
}

// Adam state sidecar <checkpoint>.adam: "GSRA", u32 version 1, u64 P, i64 step,
// f32 m[P], f32 v[P] (little-endian).
void write_adam(const std::string& path, const gsr::cuda::Context::OptimState& o) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw gsr::ResourceError("cannot write " + path);
    const std::uint32_t ver = 1;
    const std::uint64_t P = o.m.size();
    const std::int64_t st = o.step;
    f.write("GSRA", 4);
    f.write(reinterpret_cast<const char*>(&ver), 4);
    f.write(reinterpret_cast<const char*>(&P), 8);
    f.write(reinterpret_cast<const char*>(&st), 8);
    f.write(reinterpret_cast<const char*>(o.m.data()), static_cast<std::streamsize>(4 * P));
    f.write(reinterpret_cast<const char*>(o.v.data()), static_cast<std::streamsize>(4 * P));
}

bool read_adam(const std::string& path, index_t P, gsr::cuda::Context::OptimState& o) {
    std::ifstream probe(path, std::ios::binary);
    if (!probe) return false;  // parameters-only checkpoint: a warm start
    const auto b = slurp(path);
    if (b.size() < 24 || std::memcmp(b.data(), "GSRA", 4) != 0) throw gsr::FormatError(path + ": bad GSRA magic");
    if (get_le<std::uint32_t>(b, 4) != 1) throw gsr::FormatError(path + ": unsupported GSRA version");
    if (get_le<std::uint64_t>(b, 8) != static_cast<std::uint64_t>(P)) throw gsr::ShapeError(path + ": optimizer state size differs from the model");
    if (b.size() != 24 + 8 * static_cast<size_t>(P)) throw gsr::FormatError(path + ": truncated GSRA");
    o.step = get_le<std::int64_t>(b, 16);
    o.m.resize(static_cast<size_t>(P));
    o.v.resize(static_cast<size_t>(P));
    std::memcpy(o.m.data(), b.data() + 24, 4 * static_cast<size_t>(P));
    std::memcpy(o.v.data(), b.data() + 24 + 4 * static_cast<size_t>(P), 4 * static_cast<size_t>(P));
    return true;
}

// NCCL id exchange through a file (rank 0 writes it atomically, the others poll).
std::vector<unsigned char> exchange_comm_id(const std::string& path, int rank) {
    if (rank == 0) {
        const auto id = gsr::cuda::Context::comm_unique_id();
        const std::string tmp = path + ".tmp";
        {
            std::ofstream f(tmp, std::ios::binary);
            if (!f) throw gsr::ResourceError("cannot write " + tmp);
            f.write(reinterpret_cast<const char*>(id.data()), static_cast<std::streamsize>(id.size()));
        }
        if (std::rename(tmp.c_str(), path.c_str()) != 0) throw gsr::ResourceError("cannot publish " + path);
        return id;
    }
    for (int i = 0; i < 1200; ++i) {
        std::ifstream f(path, std::ios::binary);
        if (f) {
            std::vector<unsigned char> id((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
            if (id.size() == 128) return id;
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(50));
    }
    throw gsr::ResourceError("no NCCL id in " + path + " after 60 s");
}

const char* kSplitName[3] = {"train", "val", "test"};

int usage() {
    std::cerr << "usage: gsrnet-cuda train --graph G.gsrg --nodes N.gsrn [--model gsrc|gsr|baseline] [--layers L] [--hidden D]\n"
                 "                        [--groups C] [--k K] [--epochs E] [--lr LR] [--norm none|row_mean|sym]\n"
                 "                        [--precision fp32|tf32] [--seed S] [--params init.f32] [--resume in.gsrp]\n"
                 "                        [--checkpoint out.gsrp] [--report out.jsonl] [--device I] [--threads T]\n"
                 "                        [--nranks N --rank R --comm-file F]\n";
    return 1;
}

int run(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    if (cmd == "version") {
        char v[128];
        gsrc_version(v, sizeof v);
        std::cout << gsr::kArtifactVersion << " / " << v << "\n";
        return 0;
    }
    if (cmd != "train") return usage();
    std::map<std::string, std::string> a;
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw gsr::ConfigError("bad flag " + k);
        a[k.substr(2)] = argv[++i];
    }
    auto get = [&](const char* k, const std::string& d) { return a.count(k) ? a[k] : d; };
    if (!a.count("graph") || !a.count("nodes")) throw gsr::ConfigError("--graph and --nodes are required");

    gsr::cuda::NetConfig c;
    const std::string model = get("model", "gsrc");
    if (model == "gsrc") c.mode = gsr::cuda::Mode::GsrC;
    else if (model == "gsr") c.mode = gsr::cuda::Mode::Alg12;
    else if (model == "baseline") c.mode = gsr::cuda::Mode::Rev;
    else throw gsr::ConfigError("--model must be gsrc, gsr or baseline");
    c.layers = std::stoi(get("layers", "8"));
    c.hidden = std::stoi(get("hidden", "64"));
    c.groups = std::stoi(get("groups", "2"));
    c.k = std::stoi(get("k", "8"));
    const std::string prec = get("precision", "fp32");
    if (prec != "fp32" && prec != "tf32") throw gsr::ConfigError("--precision must be fp32 or tf32");
    c.precision = prec == "tf32" ? gsr::cuda::Precision::Tf32 : gsr::cuda::Precision::Fp32;
    const std::string norm_s = get("norm", "row_mean");
    gsr::cuda::Norm norm = gsr::cuda::Norm::RowMean;
    if (norm_s == "none") norm = gsr::cuda::Norm::None;
    else if (norm_s == "sym") norm = gsr::cuda::Norm::SymDegree;
    else if (norm_s != "row_mean") throw gsr::ConfigError("--norm must be none, row_mean or sym");
    const int epochs = std::stoi(get("epochs", "5"));
    gsr::cuda::OptimConfig opt;
    opt.lr = std::stof(get("lr", "1e-3"));

    const int nranks = std::stoi(get("nranks", "1")), rank = std::stoi(get("rank", "0"));
    if (nranks < 1 || rank < 0 || rank >= nranks) throw gsr::ConfigError("--rank must be in [0, --nranks)");
    if (nranks > 1 && !a.count("comm-file")) throw gsr::ConfigError("--nranks > 1 needs --comm-file");

    gsr::ThreadPool pool(std::stoi(get("threads", "0")));
    const Graph g = read_gsrg(a["graph"]);
    const Nodes d = read_gsrn(a["nodes"], &pool);
    if (d.n != g.n) throw gsr::ShapeError("node file n != graph n");
    c.d_in = static_cast<int>(d.d_in);

    gsr::cuda::Context ctx(std::stoi(get("device", nranks > 1 ? std::to_string(rank) : "0")));
    if (nranks > 1) ctx.comm_init(exchange_comm_id(a["comm-file"], rank), nranks, rank);
    ctx.upload_graph(g.n, g.row_ptr, g.col_idx, norm);
    ctx.init_model(c);
    const index_t P = ctx.num_params();
    std::vector<float> p;
    if (a.count("resume")) {
        p = read_gsrp(a["resume"], c, P);
    } else if (a.count("params")) {
        const auto b = slurp(a["params"]);
        if (b.size() != 4 * static_cast<size_t>(P)) throw gsr::ShapeError("--params: expected " + std::to_string(P) + " f32 values");
        p.resize(static_cast<size_t>(P));
        std::memcpy(p.data(), b.data(), b.size());
    } else {
        p = init_params(c, P, std::stoull(get("seed", "0")));
    }
    ctx.set_params(p);
    bool exact_resume = false;
    if (a.count("resume")) {  // Adam m, v and step from the sidecar, when the checkpoint has one
        gsr::cuda::Context::OptimState o;
        if (read_adam(a["resume"] + ".adam", P, o)) {
            ctx.set_optim_state(o);
            exact_resume = true;
        }
    }
    ctx.upload_data(d.x.data(), d.y.data(), d.train.data());
    ctx.set_graph_capture(true);

    std::ofstream rep;
    std::ostream* out = &std::cout;
    if (a.count("report")) {
        rep.open(a["report"]);
        if (!rep) throw gsr::ResourceError("cannot open report " + a["report"]);
        out = &rep;
    }
    double total = 0.0, first = 0.0, last = 0.0;
    for (int ep = 0; ep < epochs; ++ep) {
        if (ep == 1) ctx.high_water_reset();  // warmup epoch excluded
        last = ctx.train_step(opt);
        if (ep == 0) first = last;
        if (!std::isfinite(last)) throw std::runtime_error("loss is not finite at epoch " + std::to_string(ep));
        const gsrc_timing t = ctx.last_timing();
        const gsrc_mem_report m = ctx.memory();
        if (ep > 0) total += t.t_total;
        std::ostringstream s;
        s.precision(9);
        s << "{\"record\":\"epoch\",\"epoch\":" << ep << ",\"train_loss\":" << last << ",\"t_forward\":" << t.t_forward
          << ",\"t_backward\":" << t.t_backward << ",\"t_optimizer\":" << t.t_optimizer << ",\"t_copy\":" << t.t_copy << ",\"t_total\":" << t.t_total
          << ",\"peak_active_bytes\":" << m.peak_active_bytes << ",\"reserved_bytes\":" << m.reserved_bytes
          << ",\"utilization\":" << m.utilization << "}\n";
        *out << s.str();
    }
    if (a.count("checkpoint") && rank == 0) {
        write_gsrp(a["checkpoint"], ctx.params(), c);
        write_adam(a["checkpoint"] + ".adam", ctx.optim_state());
    }
    {  // CorrelationReport per split on the final predictions
        const std::vector<float> yhat = ctx.forward(g.n);
        gsr::CorrelationReport cr[3];
        gsr::parallel_for(&pool, 3, [&](index_t lo, index_t hi) {
            for (index_t sp = lo; sp < hi; ++sp) cr[sp] = gsr::correlate(yhat.data(), d.y.data(), d.split.data(), g.n, static_cast<int>(sp));
        });
        auto num = [](double v) { return std::isfinite(v) ? std::to_string(v) : std::string("null"); };
        std::ostringstream s;
        s.precision(9);
        s << "{\"record\":\"metrics\"";
        for (int sp = 0; sp < 3; ++sp)
            s << ",\"" << kSplitName[sp] << "\":{\"count\":" << cr[sp].count << ",\"pearson\":" << num(cr[sp].pearson) << ",\"spearman\":"
              << num(cr[sp].spearman) << ",\"kendall\":" << num(cr[sp].kendall) << ",\"r2\":" << num(cr[sp].r2) << "}";
        s << "}\n";
        *out << s.str();
    }
    const gsrc_mem_report m = ctx.memory();
    std::ostringstream s;
    s.precision(9);
    s << "{\"record\":\"summary\",\"version\":\"" << gsr::kArtifactVersion << "\",\"model\":\"" << model << "\",\"n\":" << g.n
      << ",\"e\":" << g.col_idx.size() << ",\"layers\":" << c.layers << ",\"hidden\":" << c.hidden << ",\"groups\":" << c.groups
      << ",\"k\":" << c.k << ",\"params\":" << P << ",\"epochs\":" << epochs << ",\"first_loss\":" << first << ",\"last_loss\":" << last
      << ",\"steps_per_s\":" << (epochs > 1 && total > 0 ? (epochs - 1) / total : 0.0) << ",\"peak_active_bytes\":" << m.peak_active_bytes
      << ",\"kernel_launches\":" << ctx.kernel_launches() << ",\"exact_resume\":" << (exact_resume ? "true" : "false")
      << ",\"nranks\":" << nranks << ",\"rank\":" << rank << ",\"host_threads\":" << pool.size() << "}\n";
    *out << s.str();
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    // Exit codes: 0 ok, 1 validation, 3 resource.
    try {
        return run(argc, argv);
    } catch (const gsr::ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return 1;
    } catch (const gsr::ResourceError& e) {
        std::cerr << "resource error: " << e.what() << "\n";
        return 3;
    } catch (const std::invalid_argument& e) {
        std::cerr << "config error: bad numeric flag value (" << e.what() << ")\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
