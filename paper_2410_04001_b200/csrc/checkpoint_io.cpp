// Checkpoint interop with the reference: the "LRNR" v1 file of
// proj/src/checkpoint.cpp -- magic, u32 version, u64 tensor count, per tensor
// (u32 name length, name, u32 rank, u64 dims, f64 data, all little endian),
// then u64 length + JSON meta (checkpoint.cpp:103-161) -- read and written
// here without a JSON library: the meta is parsed by a small recursive-descent
// parser (objects, arrays, numbers, strings, literals) and written with
// round-trip (%.17g) doubles, so files move both ways between the reference
// and this package. Tensor naming / meta keys follow put_* / get_*
// (checkpoint.cpp:163-260): lrnr.{u,v,b}.<l+1>, hyper.{w,b}.<k+1>,
// fast.{v_in,u_out,b_out,u_hat.<l+1>,b_hat.<l+1>,v_hat.<l+1>}, sampling_x.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "lrnr_gpu.h"

namespace {

thread_local std::string g_err;

// ---------------------------------------------------------------- JSON ----
struct Json {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;  // insertion order kept

    const Json& at(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return kv.second;
        throw std::runtime_error("checkpoint: meta key missing: " + k);
    }
    bool has(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return true;
        return false;
    }
    Json& set(const std::string& k) {
        for (auto& kv : obj)
            if (kv.first == k) return kv.second;
        obj.emplace_back(k, Json{});
        kind = Obj;
        return obj.back().second;
    }
    static Json number(double v) {
        Json j;
        j.kind = Num;
        j.num = v;
        return j;
    }
    static Json array_of(const std::vector<double>& v) {
        Json j;
        j.kind = Arr;
        for (double x : v) j.arr.push_back(number(x));
        return j;
    }
};

struct Parser {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
    }
    [[noreturn]] void fail(const char* what) {
        throw std::runtime_error(std::string("checkpoint: bad meta JSON (") + what + ")");
    }
    Json value() {
        ws();
        if (i >= s.size()) fail("end of input");
        const char c = s[i];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') {
            Json j;
            j.kind = Json::Str;
            j.str = string();
            return j;
        }
        if (s.compare(i, 4, "true") == 0) {
            i += 4;
            Json j;
            j.kind = Json::Bool;
            j.b = true;
            return j;
        }
        if (s.compare(i, 5, "false") == 0) {
            i += 5;
            Json j;
            j.kind = Json::Bool;
            return j;
        }
        if (s.compare(i, 4, "null") == 0) {
            i += 4;
            return Json{};
        }
        const char* beg = s.c_str() + i;
        char* end = nullptr;
        const double v = std::strtod(beg, &end);
        if (end == beg) fail("number");
        i += static_cast<size_t>(end - beg);
        return Json::number(v);
    }
    std::string string() {
        std::string out;
        ++i;  // opening quote
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                ++i;
                if (i >= s.size()) fail("escape");
                const char e = s[i];
                if (e == 'n') out += '\n';
                else if (e == 't') out += '\t';
                else if (e == 'r') out += '\r';
                else if (e == 'b') out += '\b';
                else if (e == 'f') out += '\f';
                else if (e == 'u') {
                    if (i + 4 >= s.size()) fail("\\u escape");
                    const unsigned cp = static_cast<unsigned>(std::strtoul(s.substr(i + 1, 4).c_str(), nullptr, 16));
                    if (cp < 0x80) out += static_cast<char>(cp);
                    else if (cp < 0x800) {
                        out += static_cast<char>(0xC0 | (cp >> 6));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    } else {
                        out += static_cast<char>(0xE0 | (cp >> 12));
                        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    }
                    i += 4;
                } else out += e;  // \" \\ \/
                ++i;
            } else {
                out += s[i++];
            }
        }
        if (i >= s.size()) fail("unterminated string");
        ++i;
        return out;
    }
    Json array() {
        Json j;
        j.kind = Json::Arr;
        ++i;
        ws();
        if (i < s.size() && s[i] == ']') {
            ++i;
            return j;
        }
        while (true) {
            j.arr.push_back(value());
            ws();
            if (i < s.size() && s[i] == ',') {
                ++i;
                continue;
            }
            if (i < s.size() && s[i] == ']') {
                ++i;
                return j;
            }
            fail("array");
        }
    }
    Json object() {
        Json j;
        j.kind = Json::Obj;
        ++i;
        ws();
        if (i < s.size() && s[i] == '}') {
            ++i;
            return j;
        }
        while (true) {
            ws();
            if (i >= s.size() || s[i] != '"') fail("object key");
            std::string k = string();
            ws();
            if (i >= s.size() || s[i] != ':') fail("colon");
            ++i;
            j.obj.emplace_back(std::move(k), value());
            ws();
            if (i < s.size() && s[i] == ',') {
                ++i;
                continue;
            }
            if (i < s.size() && s[i] == '}') {
                ++i;
                return j;
            }
            fail("object");
        }
    }
};

void dump(const Json& j, std::string& out) {
    char buf[64];
    switch (j.kind) {
        case Json::Null: out += "null"; break;
        case Json::Bool: out += j.b ? "true" : "false"; break;
        case Json::Num:
            if (j.num == static_cast<double>(static_cast<int64_t>(j.num)) && std::abs(j.num) < 9e15)
                std::snprintf(buf, sizeof(buf), "%lld", static_cast<long long>(j.num));
            else
                std::snprintf(buf, sizeof(buf), "%.17g", j.num);
            out += buf;
            break;
        case Json::Str:
            out += '"';
            for (char c : j.str) {
                if (c == '"' || c == '\\') {
                    out += '\\';
                    out += c;
                } else if (c == '\n') out += "\\n";
                else out += c;
            }
            out += '"';
            break;
        case Json::Arr:
            out += '[';
            for (size_t k = 0; k < j.arr.size(); ++k) {
                if (k) out += ',';
                dump(j.arr[k], out);
            }
            out += ']';
            break;
        case Json::Obj:
            out += '{';
            for (size_t k = 0; k < j.obj.size(); ++k) {
                if (k) out += ',';
                Json key;
                key.kind = Json::Str;
                key.str = j.obj[k].first;
                dump(key, out);
                out += ':';
                dump(j.obj[k].second, out);
            }
            out += '}';
            break;
    }
}

std::vector<int64_t> ints(const Json& a) {
    if (a.kind != Json::Arr) throw std::runtime_error("checkpoint: meta field is not an array");
    std::vector<int64_t> v;
    for (const Json& x : a.arr) {
        if (x.kind != Json::Num) throw std::runtime_error("checkpoint: non-numeric meta entry");
        v.push_back(static_cast<int64_t>(x.num));
    }
    return v;
}

// ---------------------------------------------------------- container ----
struct Tensor {
    std::vector<uint64_t> dims;
    std::vector<double> data;
};

}  // namespace

struct lrnr_ckpt {
    std::vector<std::pair<std::string, Tensor>> tensors;
    Json meta;

    const Tensor& find(const std::string& name) const {
        for (const auto& t : tensors)
            if (t.first == name) return t.second;
        throw std::runtime_error("checkpoint: missing tensor " + name);
    }
    void add(const std::string& name, std::vector<uint64_t> dims, const double* data) {
        uint64_t n = 1;
        for (uint64_t d : dims) n *= d;
        Tensor t;
        t.dims = std::move(dims);
        t.data.assign(data, data + n);
        for (auto& e : tensors)
            if (e.first == name) {
                e.second = std::move(t);
                return;
            }
        tensors.emplace_back(name, std::move(t));
    }
    // copies a rows x cols matrix (or a vector, cols = 0) into out; returns element count
    int64_t get(const std::string& name, uint64_t rows, uint64_t cols, double* out) const {
        const Tensor& t = find(name);
        const bool ok = cols == 0 ? (t.dims.size() == 1 && t.dims[0] == rows)
                                  : (t.dims.size() == 2 && t.dims[0] == rows && t.dims[1] == cols);
        if (!ok) throw std::runtime_error("checkpoint: tensor " + name + " has an unexpected shape");
        if (out) std::copy(t.data.begin(), t.data.end(), out);
        return static_cast<int64_t>(t.data.size());
    }
};

namespace {

uint64_t rd(std::istream& is, int bytes) {
    unsigned char buf[8];
    is.read(reinterpret_cast<char*>(buf), bytes);
    if (!is) throw std::runtime_error("checkpoint: truncated file");
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(buf[i]) << (8 * i);
    return v;
}
void wr(std::ostream& os, uint64_t v, int bytes) {
    unsigned char buf[8];
    for (int i = 0; i < bytes; ++i) buf[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xFF);
    os.write(reinterpret_cast<const char*>(buf), bytes);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return LRNR_OK;
    } catch (const std::bad_alloc&) {
        g_err = "allocation failed";
        return LRNR_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LRNR_EINVAL;
    }
}

std::string tag(int64_t k) { return std::to_string(k + 1); }

}  // namespace

extern "C" {

const char* lrnr_ckpt_last_error(void) { return g_err.c_str(); }

int lrnr_ckpt_create(lrnr_ckpt** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null argument");
        *out = new lrnr_ckpt();
        out[0]->meta.kind = Json::Obj;
    });
}

void lrnr_ckpt_free(lrnr_ckpt* c) { delete c; }

int lrnr_ckpt_load(const char* path, lrnr_ckpt** out) {
    return guarded([&] {
        if (!path || !out) throw std::invalid_argument("null argument");
        *out = nullptr;
        std::ifstream is(path, std::ios::binary);
        if (!is) throw std::runtime_error(std::string("checkpoint: cannot open ") + path);
        char magic[4];
        is.read(magic, 4);
        if (!is || std::memcmp(magic, "LRNR", 4) != 0) throw std::runtime_error("checkpoint: bad magic");
        const uint64_t version = rd(is, 4);
        if (version != 1) throw std::runtime_error("checkpoint: unsupported version " + std::to_string(version));
        auto c = std::make_unique<lrnr_ckpt>();
        const uint64_t n = rd(is, 8);
        for (uint64_t k = 0; k < n; ++k) {
            const uint64_t len = rd(is, 4);
            std::string name(len, '\0');
            is.read(name.data(), static_cast<std::streamsize>(len));
            if (!is) throw std::runtime_error("checkpoint: truncated file");
            Tensor t;
            const uint64_t rank = rd(is, 4);
            uint64_t count = 1;
            for (uint64_t d = 0; d < rank; ++d) {
                t.dims.push_back(rd(is, 8));
                count *= t.dims.back();
            }
            t.data.resize(count);
            for (uint64_t i = 0; i < count; ++i) {
                const uint64_t bits = rd(is, 8);
                std::memcpy(&t.data[i], &bits, 8);
            }
            c->tensors.emplace_back(std::move(name), std::move(t));
        }
        const uint64_t mlen = rd(is, 8);
        std::string meta(mlen, '\0');
        is.read(meta.data(), static_cast<std::streamsize>(mlen));
        if (!is) throw std::runtime_error("checkpoint: truncated file");
        Parser p{meta};
        c->meta = p.value();
        *out = c.release();
    });
}

int lrnr_ckpt_save(const lrnr_ckpt* c, const char* path) {
    return guarded([&] {
        if (!c || !path) throw std::invalid_argument("null argument");
        std::ofstream os(path, std::ios::binary);
        if (!os) throw std::runtime_error(std::string("checkpoint: cannot open ") + path + " for writing");
        os.write("LRNR", 4);
        wr(os, 1, 4);
        wr(os, c->tensors.size(), 8);
        for (const auto& e : c->tensors) {
            wr(os, e.first.size(), 4);
            os.write(e.first.data(), static_cast<std::streamsize>(e.first.size()));
            wr(os, e.second.dims.size(), 4);
            for (uint64_t d : e.second.dims) wr(os, d, 8);
            for (double x : e.second.data) {
                uint64_t bits;
                std::memcpy(&bits, &x, 8);
                wr(os, bits, 8);
            }
        }
        std::string meta;
        dump(c->meta, meta);
        wr(os, meta.size(), 8);
        os.write(meta.data(), static_cast<std::streamsize>(meta.size()));
        if (!os) throw std::runtime_error("checkpoint: write failure");
    });
}

// get_lrnr (checkpoint.cpp:175-187). Call with NULL arrays to query *L and *n_params.
int lrnr_ckpt_get_lrnr(const lrnr_ckpt* c, int* L, int64_t* widths, int64_t* ranks, int64_t* n_params,
                       double* params) {
    return guarded([&] {
        if (!c || !L || !n_params) throw std::invalid_argument("null argument");
        const Json& m = c->meta.at("lrnr");
        const std::vector<int64_t> w = ints(m.at("widths")), r = ints(m.at("ranks"));
        if (w.size() != r.size() + 1 || r.empty()) throw std::runtime_error("checkpoint: lrnr widths / ranks mismatch");
        *L = static_cast<int>(r.size());
        int64_t n = 0;
        for (size_t l = 0; l < r.size(); ++l) n += w[l + 1] * r[l] + w[l] * r[l] + w[l + 1];
        *n_params = n;
        if (widths) std::copy(w.begin(), w.end(), widths);
        if (ranks) std::copy(r.begin(), r.end(), ranks);
        if (!params) return;
        int64_t o = 0;
        for (size_t l = 0; l < r.size(); ++l) {
            o += c->get("lrnr.u." + tag(static_cast<int64_t>(l)), w[l + 1], r[l], params + o);
            o += c->get("lrnr.v." + tag(static_cast<int64_t>(l)), w[l], r[l], params + o);
            o += c->get("lrnr.b." + tag(static_cast<int64_t>(l)), w[l + 1], 0, params + o);
        }
    });
}

int lrnr_ckpt_put_lrnr(lrnr_ckpt* c, int L, const int64_t* widths, const int64_t* ranks, const double* params) {
    return guarded([&] {
        if (!c || !widths || !ranks || !params || L < 1) throw std::invalid_argument("bad argument");
        int64_t o = 0;
        std::vector<double> wv, rv;
        for (int l = 0; l <= L; ++l) wv.push_back(static_cast<double>(widths[l]));
        for (int l = 0; l < L; ++l) {
            rv.push_back(static_cast<double>(ranks[l]));
            const uint64_t mo = static_cast<uint64_t>(widths[l + 1]), mi = static_cast<uint64_t>(widths[l]),
                           r = static_cast<uint64_t>(ranks[l]);
            c->add("lrnr.u." + tag(l), {mo, r}, params + o);
            o += static_cast<int64_t>(mo * r);
            c->add("lrnr.v." + tag(l), {mi, r}, params + o);
            o += static_cast<int64_t>(mi * r);
            c->add("lrnr.b." + tag(l), {mo}, params + o);
            o += static_cast<int64_t>(mo);
        }
        Json& m = c->meta.set("lrnr");
        m.kind = Json::Obj;
        m.set("widths") = Json::array_of(wv);
        m.set("ranks") = Json::array_of(rv);
    });
}

// get_hyper (checkpoint.cpp:201-216): hw = K + 1 layer widths (hw[0] = 3),
// params in lrnr_gpu_set_hyper's flat layout (W_k row-major, then b_k).
int lrnr_ckpt_get_hyper(const lrnr_ckpt* c, int* K, int64_t* hw, int64_t* n_params, double* params, double* lo,
                        double* hi) {
    return guarded([&] {
        if (!c || !K || !n_params) throw std::invalid_argument("null argument");
        const Json& m = c->meta.at("hyper");
        const int k_layers = static_cast<int>(m.at("layers").num);
        *K = k_layers;
        std::vector<int64_t> w(static_cast<size_t>(k_layers) + 1);
        for (int k = 0; k < k_layers; ++k) {
            const Tensor& t = c->find("hyper.w." + tag(k));
            if (t.dims.size() != 2) throw std::runtime_error("checkpoint: hyper.w is not a matrix");
            w[k] = static_cast<int64_t>(t.dims[1]);
            w[k + 1] = static_cast<int64_t>(t.dims[0]);
        }
        int64_t n = 0;
        for (int k = 0; k < k_layers; ++k) n += w[k + 1] * w[k] + w[k + 1];
        *n_params = n;
        if (hw) std::copy(w.begin(), w.end(), hw);
        if (lo || hi) {
            const Json& bl = m.at("box_lo");
            const Json& bh = m.at("box_hi");
            for (int i = 0; i < 3; ++i) {
                if (lo) lo[i] = bl.arr.at(static_cast<size_t>(i)).num;
                if (hi) hi[i] = bh.arr.at(static_cast<size_t>(i)).num;
            }
        }
        if (!params) return;
        int64_t o = 0;
        for (int k = 0; k < k_layers; ++k) {
            o += c->get("hyper.w." + tag(k), w[k + 1], w[k], params + o);
            o += c->get("hyper.b." + tag(k), w[k + 1], 0, params + o);
        }
    });
}

int lrnr_ckpt_put_hyper(lrnr_ckpt* c, int K, const int64_t* hw, const double* params, int L_split,
                        const int64_t* split, const double* lo, const double* hi) {
    return guarded([&] {
        if (!c || !hw || !params || !split || !lo || !hi || K < 1) throw std::invalid_argument("bad argument");
        int64_t o = 0;
        for (int k = 0; k < K; ++k) {
            const uint64_t rows = static_cast<uint64_t>(hw[k + 1]), cols = static_cast<uint64_t>(hw[k]);
            c->add("hyper.w." + tag(k), {rows, cols}, params + o);
            o += static_cast<int64_t>(rows * cols);
            c->add("hyper.b." + tag(k), {rows}, params + o);
            o += static_cast<int64_t>(rows);
        }
        std::vector<double> sp;
        for (int l = 0; l < L_split; ++l) sp.push_back(static_cast<double>(split[l]));
        Json& m = c->meta.set("hyper");
        m.kind = Json::Obj;
        m.set("layers") = Json::number(K);
        m.set("split") = Json::array_of(sp);
        m.set("box_lo") = Json::array_of({lo[0], lo[1], lo[2]});
        m.set("box_hi") = Json::array_of({hi[0], hi[1], hi[2]});
    });
}

int lrnr_ckpt_has_fast(const lrnr_ckpt* c) { return c && c->meta.kind == Json::Obj && c->meta.has("fast") ? 1 : 0; }

// get_fast (checkpoint.cpp:231-246): params in lrnr_gpu_set_fast's flat layout
// (v_in, per inner layer u_hat, b_hat, v_hat, then u_out, b_out).
int lrnr_ckpt_get_fast(const lrnr_ckpt* c, int* L, int64_t* ranks, int64_t* red_ranks, int64_t* n_params,
                       double* params) {
    return guarded([&] {
        if (!c || !L || !n_params) throw std::invalid_argument("null argument");
        const Json& m = c->meta.at("fast");
        const std::vector<int64_t> r = ints(m.at("ranks")), h = ints(m.at("red_ranks"));
        if (r.size() != h.size() + 1) throw std::runtime_error("checkpoint: fast ranks / red_ranks mismatch");
        *L = static_cast<int>(r.size());
        const Tensor& vin = c->find("fast.v_in");
        const Tensor& uout = c->find("fast.u_out");
        if (vin.dims.size() != 2 || uout.dims.size() != 2) throw std::runtime_error("checkpoint: fast shapes");
        const int64_t m_in = static_cast<int64_t>(vin.dims[0]), m_out = static_cast<int64_t>(uout.dims[0]);
        int64_t n = m_in * r[0] + m_out * r.back() + m_out;
        for (size_t l = 0; l + 1 < r.size(); ++l) n += h[l] * r[l] + h[l] + h[l] * r[l + 1];
        *n_params = n;
        if (ranks) std::copy(r.begin(), r.end(), ranks);
        if (red_ranks) std::copy(h.begin(), h.end(), red_ranks);
        if (!params) return;
        int64_t o = c->get("fast.v_in", m_in, r[0], params);
        for (size_t l = 0; l + 1 < r.size(); ++l) {
            const int64_t ll = static_cast<int64_t>(l);
            o += c->get("fast.u_hat." + tag(ll), h[l], r[l], params + o);
            o += c->get("fast.b_hat." + tag(ll), h[l], 0, params + o);
            o += c->get("fast.v_hat." + tag(ll), h[l], r[l + 1], params + o);
        }
        o += c->get("fast.u_out", m_out, r.back(), params + o);
        c->get("fast.b_out", m_out, 0, params + o);
    });
}

int lrnr_ckpt_put_fast(lrnr_ckpt* c, int L, const int64_t* ranks, const int64_t* red_ranks, int64_t m_in,
                       int64_t m_out, const double* params) {
    return guarded([&] {
        if (!c || !ranks || !red_ranks || !params || L < 2) throw std::invalid_argument("bad argument");
        auto u = [](int64_t v) { return static_cast<uint64_t>(v); };
        int64_t o = 0;
        c->add("fast.v_in", {u(m_in), u(ranks[0])}, params);
        o += m_in * ranks[0];
        std::vector<std::pair<std::string, std::pair<std::vector<uint64_t>, int64_t>>> inner;
        for (int l = 0; l + 1 < L; ++l) {
            c->add("fast.u_hat." + tag(l), {u(red_ranks[l]), u(ranks[l])}, params + o);
            o += red_ranks[l] * ranks[l];
            c->add("fast.b_hat." + tag(l), {u(red_ranks[l])}, params + o);
            o += red_ranks[l];
            c->add("fast.v_hat." + tag(l), {u(red_ranks[l]), u(ranks[l + 1])}, params + o);
            o += red_ranks[l] * ranks[l + 1];
        }
        c->add("fast.u_out", {u(m_out), u(ranks[L - 1])}, params + o);
        o += m_out * ranks[L - 1];
        c->add("fast.b_out", {u(m_out)}, params + o);
        std::vector<double> rv, hv;
        for (int l = 0; l < L; ++l) rv.push_back(static_cast<double>(ranks[l]));
        for (int l = 0; l + 1 < L; ++l) hv.push_back(static_cast<double>(red_ranks[l]));
        Json& m = c->meta.set("fast");
        m.kind = Json::Obj;
        m.set("ranks") = Json::array_of(rv);
        m.set("red_ranks") = Json::array_of(hv);
    });
}

// get_sampling / put_sampling (checkpoint.cpp:262-274): X as n (x, t) pairs.
int lrnr_ckpt_get_sampling(const lrnr_ckpt* c, int64_t* n, double* xt) {
    return guarded([&] {
        if (!c || !n) throw std::invalid_argument("null argument");
        const Json& a = c->meta.at("sampling_x");
        *n = static_cast<int64_t>(a.arr.size());
        if (!xt) return;
        for (size_t i = 0; i < a.arr.size(); ++i) {
            xt[2 * i] = a.arr[i].arr.at(0).num;
            xt[2 * i + 1] = a.arr[i].arr.at(1).num;
        }
    });
}

int lrnr_ckpt_put_sampling(lrnr_ckpt* c, int64_t n, const double* xt) {
    return guarded([&] {
        if (!c || (n && !xt)) throw std::invalid_argument("bad argument");
        Json& a = c->meta.set("sampling_x");
        a = Json{};
        a.kind = Json::Arr;
        for (int64_t i = 0; i < n; ++i) a.arr.push_back(Json::array_of({xt[2 * i], xt[2 * i + 1]}));
    });
}

}  // extern "C"
