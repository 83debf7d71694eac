// capi.cpp -- the extern "C" boundary (include/tempo_b200.h): argument
// checks that mirror the reference's exceptions, the v1 GELU table parser
// and its device form, host mask streams, stash accounting, and the kernel
// launches.  No allocation, no hidden synchronization (except the explicitly
// synchronous tempo_ln_check_gamma).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "tempo_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return TEMPO_OK;
    return fail(TEMPO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                    cudaGetErrorString(e) + ")");
}

cudaStream_t S(tempo_stream_t s) { return static_cast<cudaStream_t>(s); }

std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

// ---- v1 table (gelu_table.hpp:27-91, gelu_table.cpp) ---------------------
struct Segment {
    int branch = 1;
    double lo = 0.0, hi = 0.0;
    bool sqrt_shift = false;
    std::vector<double> coeffs;
};

struct ParseFail {
    std::string msg;
};

double parse_double(const std::string& tok) {  // gelu_table.cpp:23-31
    const char* begin = tok.c_str();
    char* end = nullptr;
    double v = std::strtod(begin, &end);
    if (end != begin + tok.size() || tok.empty()) throw ParseFail{"bad number '" + tok + "' in table"};
    return v;
}

double parse_kv(const std::string& tok, const std::string& key) {  // :34-41
    std::string prefix = key + "=";
    if (tok.rfind(prefix, 0) != 0)
        throw ParseFail{"expected '" + key + "=...' in table header, got '" + tok + "'"};
    return parse_double(tok.substr(prefix.size()));
}

}  // namespace

struct tempo_gelu_table_s {
    double x_star = 0.0, y_min = 0.0, tol = 0.0, max_err = -1.0;
    std::vector<Segment> seg[2];  // ascending lo
    tb::GeluDevTable dev;
    bool dev_ok = false;  // within the device limits (kMaxSeg, kMaxCoef)
    bool verified() const { return max_err >= 0.0; }

    // GeluPolyTable::eval (gelu_table.cpp:172-188) in double.
    double eval(double y, int m) const {
        if (m == 0) {
            if (y >= 0.0) return 0.0;
            if (y < y_min) y = y_min;
        } else if (y < y_min) {
            y = y_min;
        }
        const auto& s = seg[m];
        std::size_t lo = 0, hi = s.size();
        while (hi - lo > 1) {
            std::size_t mid = (lo + hi) / 2;
            if (s[mid].lo <= y) lo = mid; else hi = mid;
        }
        const Segment& g = s[lo];
        if (g.coeffs.size() == 1) return g.coeffs[0];
        double u, ulo, uhi;
        if (g.sqrt_shift) {
            u = std::sqrt(std::max(y - y_min, 0.0));
            ulo = std::sqrt(std::max(g.lo - y_min, 0.0));
            uhi = std::sqrt(g.hi - y_min);
        } else {
            u = y;
            ulo = g.lo;
            uhi = g.hi;
        }
        double t = std::clamp(2.0 * (u - ulo) / (uhi - ulo) - 1.0, -1.0, 1.0);
        double b1 = 0.0, b2 = 0.0;
        for (std::size_t k = g.coeffs.size(); k-- > 1;) {
            double b = 2.0 * t * b1 - b2 + g.coeffs[k];
            b2 = b1;
            b1 = b;
        }
        return t * b1 - b2 + g.coeffs[0];
    }
};

namespace {

// Smallest float >= v / > v (exact fp32 stand-ins for double comparisons).
float float_up(double v) {
    float f = (float)v;
    if ((double)f < v) f = std::nextafter(f, std::numeric_limits<float>::infinity());
    return f;
}
float float_above(double v) {
    float f = float_up(v);
    if ((double)f == v) f = std::nextafter(f, std::numeric_limits<float>::infinity());
    return f;
}

void validate_tiling(const tempo_gelu_table_s& t) {  // gelu_table.cpp:106-148
    if (t.seg[0].empty() || t.seg[1].empty()) throw ParseFail{"table must cover both branches"};
    auto chain = [&](const std::vector<Segment>& segs, int branch, double lo_expect,
                     double hi_expect) {
        double cursor = lo_expect;
        for (const Segment& s : segs) {
            if (s.lo != cursor)
                throw ParseFail{"branch " + std::to_string(branch) + " segments leave a gap at " +
                                g17(cursor)};
            if (!(s.lo < s.hi)) throw ParseFail{"segment bounds not increasing at " + g17(s.lo)};
            if (s.coeffs.empty() || s.coeffs.size() > 64)
                throw ParseFail{"segment coefficient count out of range"};
            for (double c : s.coeffs)
                if (!std::isfinite(c)) throw ParseFail{"non-finite coefficient in table"};
            if (!std::isfinite(s.hi) && s.coeffs.size() != 1)
                throw ParseFail{"unbounded segment must be constant"};
            if (s.sqrt_shift && s.lo != t.y_min)
                throw ParseFail{"sqrt-shift segment must start at the minimum"};
            cursor = s.hi;
        }
        if (cursor != hi_expect)
            throw ParseFail{"branch " + std::to_string(branch) + " does not reach " +
                            g17(hi_expect)};
    };
    chain(t.seg[0], 0, t.y_min, 0.0);
    chain(t.seg[1], 1, t.y_min, std::numeric_limits<double>::infinity());
}

// Chebyshev series on [-1, 1] -> power-basis coefficients (fp64).
std::vector<double> cheb_to_mono(const std::vector<double>& c) {
    const std::size_t n = c.size();
    std::vector<double> out(n, 0.0), tkm1(n, 0.0), tk(n, 0.0);
    tkm1[0] = 1.0;  // T_0
    if (n > 1) tk[1] = 1.0;  // T_1
    for (std::size_t k = 0; k < n; ++k) {
        const std::vector<double>& T = k == 0 ? tkm1 : tk;
        for (std::size_t j = 0; j < n; ++j) out[j] += c[k] * T[j];
        if (k >= 1 && k + 1 < n) {  // T_{k+1} = 2t T_k - T_{k-1}
            std::vector<double> nx(n, 0.0);
            for (std::size_t j = 0; j + 1 < n; ++j) nx[j + 1] += 2.0 * tk[j];
            for (std::size_t j = 0; j < n; ++j) nx[j] -= tkm1[j];
            tkm1 = tk;
            tk = nx;
        }
    }
    return out;
}

void build_device(tempo_gelu_table_s& t) {
    tb::GeluDevTable& d = t.dev;
    std::memset(&d, 0, sizeof(d));
    // The device table appends one segment to branch 0: [0, +inf) with the
    // constant 0, which is eval's "m = 0 and y >= 0 -> 0" rule
    // (gelu_table.cpp:182) expressed as a segment, so the kernel needs no
    // special case.
    const int n0 = (int)t.seg[0].size() + 1, n1 = (int)t.seg[1].size();
    int ncoef = 1;
    for (int b = 0; b < 2; ++b)
        for (const Segment& s : t.seg[b]) ncoef = std::max(ncoef, (int)s.coeffs.size());
    t.dev_ok = n0 + n1 <= tb::kMaxSeg && ncoef <= tb::kMaxCoef;
    if (!t.dev_ok) return;
    d.xstar_gt = float_above(t.x_star);
    d.ymin_up = float_up(t.y_min);
    d.ymin_hi = (float)t.y_min;
    d.ymin_lo = (float)(t.y_min - (double)d.ymin_hi);
    d.nseg[0] = n0;
    d.nseg[1] = n1;
    d.ncoef = ncoef;
    d.stride = ncoef | 1;
    // Horner in the power basis when its error bound (coefficient rounding +
    // Horner's (2d)eps sum|a_k|, t in [-1, 1]) stays below 4e-6; the default
    // fit's bound is 1.7e-6 (measured 1.2e-7), else Clenshaw as the reference.
    bool horner = ncoef <= 16;
    Segment zero;
    zero.branch = 0;
    zero.lo = 0.0;
    zero.hi = std::numeric_limits<double>::infinity();
    zero.coeffs = {0.0};
    int k = 0;
    for (int b = 0; b < 2; ++b) {
        std::vector<const Segment*> segs;
        for (const Segment& s : t.seg[b]) segs.push_back(&s);
        if (b == 0) segs.push_back(&zero);
        for (const Segment* sp : segs) {
            const Segment& s = *sp;
            d.lo_up[k] = float_up(s.lo);
            d.sqrt_shift[k] = s.sqrt_shift ? 1 : 0;
            double sc = 0.0, u0 = 0.0;  // t = sc * (u - u0)
            if (s.coeffs.size() == 1) {
                d.s[k] = 0.0f;
                d.b[k] = 0.0f;
            } else {
                double ulo, uhi;
                if (s.sqrt_shift) {
                    ulo = std::sqrt(std::max(s.lo - t.y_min, 0.0));
                    uhi = std::sqrt(s.hi - t.y_min);
                } else {
                    ulo = s.lo;
                    uhi = s.hi;
                }
                sc = 2.0 / (uhi - ulo);
                u0 = 0.5 * (uhi + ulo);
                d.s[k] = (float)sc;
                d.b[k] = (float)(-(uhi + ulo) / (uhi - ulo));
                if (d.s[k] == 0.0f) d.s[k] = std::numeric_limits<float>::min();
            }
            for (std::size_t c = 0; c < s.coeffs.size(); ++c) d.coef[k][c] = (float)s.coeffs[c];
            if (s.coeffs.size() <= 15) {
                // power basis of t, then of v = u - u0 with t = sc * v:
                // a'_k = a_k * sc^k; |sc * v| <= 1 inside the segment, so
                // Horner's bound in v is the one in t
                std::vector<double> a = cheb_to_mono(s.coeffs);
                double suma = 0.0, sumd = 0.0, sk = 1.0;
                d.u0[k] = (float)u0;
                for (std::size_t c = 0; c < a.size(); ++c) {
                    const double ak = a[c] * sk;
                    d.monov[k][c] = (float)ak;
                    if (!std::isfinite(d.monov[k][c]) ||
                        (ak != 0.0 && std::abs(ak) < (double)std::numeric_limits<float>::min()))
                        horner = false;
                    sk *= sc;
                    suma += std::abs(a[c]);
                    sumd += (double)c * std::abs(a[c]);  // bounds |p'(t)| on [-1, 1]
                }
                // Horner's (2d+2)eps sum|a_k|, plus the fp32 roundings of u
                // and u0 (each <= eps |u|) moved through t = sc * v
                const double umax = std::abs(u0) + (sc > 0.0 ? 1.0 / sc : 0.0);
                if (suma * (2.0 * (double)a.size() + 2.0) * 0x1p-24 +
                        sumd * sc * 2.0 * umax * 0x1p-24 > 4e-6)
                    horner = false;
            } else {
                horner = false;
            }
            ++k;
        }
    }
    d.horner = horner ? 1 : 0;
}

tempo_gelu_table_s* parse_table(const std::string& text) {  // gelu_table.cpp:227-301
    std::istringstream in(text);
    std::string line;
    if (!std::getline(in, line)) throw ParseFail{"empty table input"};
    std::istringstream hdr(line);
    std::string magic, version, tok;
    hdr >> magic >> version;
    if (magic != "gelu-poly-table") throw ParseFail{"not a gelu-poly-table file"};
    if (version != "v1") throw ParseFail{"unsupported table version '" + version + "'"};
    auto* t = new tempo_gelu_table_s();
    try {
        if (!(hdr >> tok)) throw ParseFail{"truncated table header"};
        t->x_star = parse_kv(tok, "x_star");
        if (!(hdr >> tok)) throw ParseFail{"truncated table header"};
        t->y_min = parse_kv(tok, "y_min");
        if (!(hdr >> tok)) throw ParseFail{"truncated table header"};
        t->tol = parse_kv(tok, "tol");
        if (!(hdr >> tok)) throw ParseFail{"truncated table header"};
        double max_err = parse_kv(tok, "max_err");
        if (hdr >> tok) throw ParseFail{"unexpected token '" + tok + "' in table header"};
        while (std::getline(in, line)) {
            std::istringstream ls(line);
            std::vector<std::string> toks;
            while (ls >> tok) toks.push_back(tok);
            if (toks.empty()) continue;
            if (toks.size() < 6) throw ParseFail{"malformed segment line '" + line + "'"};
            Segment s;
            if (toks[0] == "0") s.branch = 0;
            else if (toks[0] == "1") s.branch = 1;
            else throw ParseFail{"segment branch must be 0 or 1, got '" + toks[0] + "'"};
            s.lo = parse_double(toks[1]);
            s.hi = parse_double(toks[2]);
            if (toks[3] == "direct-y") s.sqrt_shift = false;
            else if (toks[3] == "sqrt-shift") s.sqrt_shift = true;
            else throw ParseFail{"unknown segment variable '" + toks[3] + "'"};
            long degree = 0;
            {
                const char* b = toks[4].c_str();
                char* e = nullptr;
                errno = 0;
                degree = std::strtol(b, &e, 10);
                if (e == b || *e != '\0' || errno == ERANGE)
                    throw ParseFail{"bad segment degree '" + toks[4] + "'"};
            }
            if (degree < 0 || toks.size() != 6 + static_cast<std::size_t>(degree))
                throw ParseFail{"segment degree " + std::to_string(degree) +
                                " does not match coefficient count"};
            for (std::size_t i = 5; i < toks.size(); ++i) s.coeffs.push_back(parse_double(toks[i]));
            t->seg[s.branch].push_back(std::move(s));
        }
        // GeluPolyTable(minimum, tolerance, segments) (gelu_table.cpp:83-104)
        if (!(t->tol > 0.0)) throw ParseFail{"table tolerance must be positive"};
        auto by_lo = [](const Segment& a, const Segment& b) { return a.lo < b.lo; };
        std::sort(t->seg[0].begin(), t->seg[0].end(), by_lo);
        std::sort(t->seg[1].begin(), t->seg[1].end(), by_lo);
        validate_tiling(*t);
        if (max_err >= 0.0) t->max_err = max_err;  // :300
    } catch (...) {
        delete t;
        throw;
    }
    build_device(*t);
    return t;
}

// The default fit (fit::fit_table(), gelu_fit.cpp:331-382, default
// FitOptions), exactly as the reference serializes it; regenerate with
// tests/golden/make_golden.py (tests/test_golden.py pins equality).
const char* kDefaultTable =
    "gelu-poly-table v1 x_star=-0.75179152469399924 y_min=-0.16997120747990366 tol=0.0001 "
    "max_err=7.9034905239312725e-05\n"
    "0 -0.16997120747990366 -0.12747840560992774 sqrt-shift 3 -0.071964327147487822 "
    "-0.063189101190441424 0.0093155715388479159 0.00056566659241474209\n"
    "0 -0.12747840560992774 -0.063739202804963868 direct-y 3 -0.12073442364168202 "
    "0.010279259520732316 0.0053991795546408372 -0.00030552209372212605\n"
    "0 -0.063739202804963868 0 direct-y 10 -0.059840943034316356 0.051390230368853047 "
    "0.0066086341265260183 0.0009559203167106619 0.00038570630410708406 "
    "0.00017917921758346382 9.8533855290003819e-05 5.9603676026244355e-05 "
    "3.8704338519361889e-05 2.6495497882348027e-05 1.8900427578820303e-05\n"
    "1 -0.16997120747990366 1.8725215943900724 sqrt-shift 6 0.69354245105000201 "
    "0.58950164648434789 -0.1591178885804177 -0.044684065878817986 0.011744517239509158 "
    "0.001875575973017973 0.00051826019516842525\n"
    "1 1.8725215943900724 8 direct-y 9 1.017348155224377 -0.031662194028806913 "
    "0.023877168977438669 -0.014456922843931699 0.0064794394932634111 "
    "-0.0015253109477308851 -0.00055213912790641213 0.00085695970436623203 "
    "-0.00051143919664118091 0.00016352762911376676\n"
    "1 8 inf direct-y 0 1\n";

int check_p(double p) {  // ops_reference.cpp:148-151
    if (!(p >= 0.0) || p >= 1.0)
        return fail(TEMPO_ERR_PARAM, "dropout p must lie in [0, 1), got " + std::to_string(p));
    return TEMPO_OK;
}

// keep <=> u >= p with u = r * 2^-32  <=>  r >= ceil(p * 2^32).
uint64_t philox_threshold(double p) { return (uint64_t)std::ceil(p * 4294967296.0); }

int check_mode(tempo_mask_mode_t mode) {
    if (mode != TEMPO_MASK_SUPPLIED && mode != TEMPO_MASK_PHILOX)
        return fail(TEMPO_ERR_PARAM, "unknown mask mode " + std::to_string((int)mode));
    return TEMPO_OK;
}

int check_n(int64_t n, const char* what) {
    if (n < 0) return fail(TEMPO_ERR_DIMENSION, std::string(what) + ": negative element count");
    return TEMPO_OK;
}

int check_rows(int64_t rows, int64_t cols, const char* what) {
    if (rows < 0 || cols < 0)
        return fail(TEMPO_ERR_DIMENSION, std::string(what) + ": negative shape");
    if (cols == 0 && rows > 0)
        return fail(TEMPO_ERR_DIMENSION, std::string(what) + " over empty last dim");
    return TEMPO_OK;
}

}  // namespace

namespace tb {

int grid_for(const void* kernel, int block, size_t smem, int64_t work_items, int cap_per_sm,
             int waves) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
    static std::map<std::pair<int, const void*>, bool> optin;  // per (device, kernel)
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0, sms = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        // The dynamic-smem limit is a per-KERNEL attribute: raise it once to
        // the device's opt-in maximum, so launches of the same kernel with
        // different dynamic sizes never see a stale smaller limit (static +
        // dynamic may exceed the 48 KB default even when dynamic alone does not).
        if (smem > 0 && !optin[{dev, kernel}]) {
            int maxopt = 0;
            cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kernel);
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 maxopt - (int)fa.sharedSizeBytes);
            optin[{dev, kernel}] = true;
        }
        auto key = std::make_tuple(dev, kernel, block, smem);
        auto it = cache.find(key);
        if (it != cache.end()) {
            per_sm = it->second & 0xffff;
            sms = it->second >> 16;
        } else {
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
            if (per_sm < 1) per_sm = 1;
            if (sms < 1) sms = 1;
            cache[key] = per_sm | (sms << 16);
        }
    }
    if (cap_per_sm > 0 && per_sm > cap_per_sm) per_sm = cap_per_sm;
    int64_t full = (int64_t)per_sm * sms * (waves > 1 ? waves : 1);
    if (work_items < 1) work_items = 1;
    return (int)std::min<int64_t>(full, work_items);
}

}  // namespace tb

extern "C" {

const char* tempo_last_error(void) { return g_err.c_str(); }
const char* tempo_version(void) { return "tempo-b200 0.1.0 (sm_100a)"; }

// ---- table -----------------------------------------------------------------
int tempo_gelu_table_create(const char* v1_text, tempo_gelu_table_t* out) {
    if (!out) return fail(TEMPO_ERR_PARAM, "null output handle");
    *out = nullptr;
    if (!v1_text) return fail(TEMPO_ERR_PARSE, "empty table input");
    try {
        *out = parse_table(v1_text);
    } catch (const ParseFail& e) {
        return fail(TEMPO_ERR_PARSE, e.msg);
    } catch (const std::exception& e) {
        return fail(TEMPO_ERR_UNKNOWN, e.what());
    }
    return TEMPO_OK;
}

int tempo_gelu_table_destroy(tempo_gelu_table_t table) {
    delete table;
    return TEMPO_OK;
}

int tempo_gelu_table_info(tempo_gelu_table_t t, double* x_star, double* y_min, double* tolerance,
                          double* verified_max_error, int* verified, int* n_segments,
                          int* max_degree) {
    if (!t) return fail(TEMPO_ERR_CONFIG, "null table");
    if (x_star) *x_star = t->x_star;
    if (y_min) *y_min = t->y_min;
    if (tolerance) *tolerance = t->tol;
    if (verified_max_error) *verified_max_error = t->max_err;
    if (verified) *verified = t->verified() ? 1 : 0;
    int deg = 0;
    for (int b = 0; b < 2; ++b)
        for (const Segment& s : t->seg[b]) deg = std::max(deg, (int)s.coeffs.size() - 1);
    if (n_segments) *n_segments = (int)(t->seg[0].size() + t->seg[1].size());
    if (max_degree) *max_degree = deg;
    return TEMPO_OK;
}

int tempo_gelu_table_serialize(tempo_gelu_table_t t, char* buf, size_t cap, size_t* len) {
    if (!t) return fail(TEMPO_ERR_CONFIG, "null table");
    std::ostringstream os;  // gelu_table.cpp:204-218
    os << "gelu-poly-table v1 x_star=" << g17(t->x_star) << " y_min=" << g17(t->y_min)
       << " tol=" << g17(t->tol) << " max_err=" << g17(t->max_err) << "\n";
    for (int b = 0; b < 2; ++b) {
        for (const Segment& s : t->seg[b]) {
            os << s.branch << ' ' << g17(s.lo) << ' ' << g17(s.hi) << ' '
               << (s.sqrt_shift ? "sqrt-shift" : "direct-y") << ' ' << s.coeffs.size() - 1;
            for (double c : s.coeffs) os << ' ' << g17(c);
            os << "\n";
        }
    }
    std::string str = os.str();
    if (len) *len = str.size();
    if (buf && cap > str.size()) std::memcpy(buf, str.c_str(), str.size() + 1);
    return TEMPO_OK;
}

const char* tempo_gelu_default_table_v1(void) { return kDefaultTable; }

int tempo_gelu_table_eval_host(tempo_gelu_table_t t, const double* y, const uint8_t* m,
                               double* out, int64_t n) {
    if (!t) return fail(TEMPO_ERR_CONFIG, "eval on an empty table");
    for (int64_t i = 0; i < n; ++i) {
        if (m[i] > 1) return fail(TEMPO_ERR_PARAM, "branch flag must be 0 or 1");
        out[i] = t->eval(y[i], m[i]);
    }
    return TEMPO_OK;
}

// ---- GELU --------------------------------------------------------------------
int tempo_gelu_ip_fwd(const float* x, float* y, uint32_t* mask, int64_t n,
                      tempo_gelu_table_t table, tempo_stream_t stream) {
    if (!table) return fail(TEMPO_ERR_CONFIG, "in-place gelu needs a fitted table");
    if (int rc = check_n(n, "gelu")) return rc;
    if (n > 0 && (!x || !y || !mask)) return fail(TEMPO_ERR_PARAM, "gelu: null tensor pointer");
    return cuda_status(tb::launch_gelu_fwd(x, y, mask, n, table->dev.xstar_gt, S(stream)),
                       "tempo_gelu_ip_fwd");
}

int tempo_gelu_ip_fwd_exact(const float* x, float* y, uint32_t* mask, int64_t n,
                            tempo_gelu_table_t table, tempo_stream_t stream) {
    if (!table) return fail(TEMPO_ERR_CONFIG, "in-place gelu needs a fitted table");
    if (int rc = check_n(n, "gelu")) return rc;
    if (n > 0 && (!x || !y || !mask)) return fail(TEMPO_ERR_PARAM, "gelu: null tensor pointer");
    return cuda_status(tb::launch_gelu_fwd_exact(x, y, mask, n, table->dev.xstar_gt, S(stream)),
                       "tempo_gelu_ip_fwd_exact");
}

int tempo_gelu_ip_bwd(const float* dy, const float* y, const uint32_t* mask,
                      tempo_gelu_table_t table, float* dx, int64_t n, tempo_stream_t stream) {
    if (!table) return fail(TEMPO_ERR_CONFIG, "in-place gelu needs a fitted table");
    if (!table->verified())  // ops_tempo.cpp:80-83
        return fail(TEMPO_ERR_CONFIG, "gelu backward requires a sweep-verified table");
    if (!table->dev_ok)
        return fail(TEMPO_ERR_UNSUPPORTED, "table exceeds the device limits (32 segments)");
    if (int rc = check_n(n, "gelu")) return rc;
    if (n > 0 && (!dy || !y || !mask || !dx))
        return fail(TEMPO_ERR_PARAM, "gelu: null tensor pointer");
    return cuda_status(tb::launch_gelu_bwd(dy, y, mask, table->dev, dx, n, S(stream)),
                       "tempo_gelu_ip_bwd");
}

// ---- LayerNorm -----------------------------------------------------------------
int tempo_ln_ip_fwd(const float* x, const float* gamma, const float* beta, double eps, float* y,
                    float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                    tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "row_moments")) return rc;
    if (!(eps > 0.0)) return fail(TEMPO_ERR_PARAM, "layernorm epsilon must be positive");
    if (rows > 0 && (!x || !gamma || !beta || !y || !rstd))
        return fail(TEMPO_ERR_PARAM, "layernorm: null tensor pointer");
    if (cols > std::numeric_limits<int>::max())
        return fail(TEMPO_ERR_DIMENSION, "layernorm: row too long");
    return cuda_status(
        tb::launch_ln_fwd(x, gamma, beta, eps, y, rstd, rows, cols, dev_status, S(stream)),
        "tempo_ln_ip_fwd");
}

int tempo_ln_check_gamma(const float* gamma, int64_t cols, tempo_stream_t stream) {
    if (cols < 0) return fail(TEMPO_ERR_DIMENSION, "negative column count");
    std::vector<float> h((size_t)cols);
    if (cols > 0) {
        cudaError_t e = cudaMemcpyAsync(h.data(), gamma, cols * sizeof(float),
                                        cudaMemcpyDeviceToHost, S(stream));
        if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
        if (e != cudaSuccess) return cuda_status(e, "tempo_ln_check_gamma");
    }
    for (int64_t j = 0; j < cols; ++j) {
        if (std::abs((double)h[j]) < 1e-12)  // ops_tempo.cpp:100-106, ops_tempo.hpp:46
            return fail(TEMPO_ERR_PARAM, "layernorm gamma[" + std::to_string(j) +
                                             "] too close to zero to invert the output");
    }
    return TEMPO_OK;
}

size_t tempo_ln_ip_bwd_workspace_size(int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return 0;
    return tb::ln_bwd_workspace(rows, cols);
}

int tempo_ln_ip_bwd(const float* dy, const float* y, const float* rstd, const float* gamma,
                    const float* beta, float* dx, float* dgamma, float* dbeta, void* workspace,
                    size_t workspace_bytes, int64_t rows, int64_t cols, tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "layernorm backward")) return rc;
    if (cols > std::numeric_limits<int>::max())
        return fail(TEMPO_ERR_DIMENSION, "layernorm: row too long");
    if (cols > 0 && (!gamma || !beta || !dgamma || !dbeta))
        return fail(TEMPO_ERR_PARAM, "layernorm: null parameter pointer");
    if (rows > 0 && (!dy || !y || !rstd || !dx))
        return fail(TEMPO_ERR_PARAM, "layernorm: null tensor pointer");
    size_t need = tempo_ln_ip_bwd_workspace_size(rows, cols);
    if (workspace_bytes < need || (need > 0 && !workspace))
        return fail(TEMPO_ERR_PARAM, "layernorm backward workspace too small: need " +
                                         std::to_string(need) + " bytes");
    return cuda_status(tb::launch_ln_bwd(dy, y, rstd, gamma, beta, dx, dgamma, dbeta, workspace,
                                         rows, cols, S(stream)),
                       "tempo_ln_ip_bwd");
}

int tempo_ln_ip_bwd_partials(const float* dy, const float* y, const float* rstd,
                             const float* gamma, const float* beta, float* dx, void* workspace,
                             size_t workspace_bytes, int64_t rows, int64_t cols, int64_t* nparts,
                             tempo_stream_t stream) {
    if (!nparts) return fail(TEMPO_ERR_PARAM, "layernorm: null nparts");
    *nparts = 0;
    if (int rc = check_rows(rows, cols, "layernorm backward")) return rc;
    if (cols > std::numeric_limits<int>::max())
        return fail(TEMPO_ERR_DIMENSION, "layernorm: row too long");
    if (cols > 0 && (!gamma || !beta)) return fail(TEMPO_ERR_PARAM, "layernorm: null parameter pointer");
    if (rows > 0 && (!dy || !y || !rstd || !dx))
        return fail(TEMPO_ERR_PARAM, "layernorm: null tensor pointer");
    size_t need = tempo_ln_ip_bwd_workspace_size(rows, cols);
    if (workspace_bytes < need || (need > 0 && !workspace))
        return fail(TEMPO_ERR_PARAM, "layernorm backward workspace too small: need " +
                                         std::to_string(need) + " bytes");
    return cuda_status(tb::launch_ln_bwd(dy, y, rstd, gamma, beta, dx, nullptr, nullptr, workspace,
                                         rows, cols, S(stream), nullptr, nullptr, 1.0, nullptr,
                                         nparts),
                       "tempo_ln_ip_bwd_partials");
}

int tempo_ln_param_reduce(const double* partials, int64_t nparts, int64_t cols, float* dgamma,
                          float* dbeta, tempo_stream_t stream) {
    if (nparts < 0 || cols < 0) return fail(TEMPO_ERR_DIMENSION, "ln_param_reduce: negative size");
    if (cols > std::numeric_limits<int>::max() / 2 || nparts > std::numeric_limits<int>::max())
        return fail(TEMPO_ERR_DIMENSION, "ln_param_reduce: too large");
    if (cols > 0 && (!dgamma || !dbeta || (nparts > 0 && !partials)))
        return fail(TEMPO_ERR_PARAM, "ln_param_reduce: null pointer");
    return cuda_status(tb::launch_ln_param_reduce(partials, nparts, cols, dgamma, dbeta, S(stream)),
                       "tempo_ln_param_reduce");
}

// ---- multi-GPU: stage 2 fused with the cross-rank sum --------------------------------
size_t tempo_ln_peer_inbox_bytes(int32_t world, int64_t cols) {
    return world > 0 && cols > 0 ? tb::ln_peer_inbox_bytes(world, cols) : 0;
}
size_t tempo_ln_peer_flag_bytes(int32_t world, int64_t cols) {
    return world > 0 && cols > 0 ? tb::ln_peer_flag_bytes(world, cols) : 0;
}

static int check_peer(const tempo_ln_peer_t* peer) {
    if (!peer) return fail(TEMPO_ERR_PARAM, "peer group: null");
    if (peer->world < 1 || peer->rank < 0 || peer->rank >= peer->world)
        return fail(TEMPO_ERR_PARAM, "peer group: bad rank/world");
    if (!peer->inbox || !peer->flags || !peer->status)
        return fail(TEMPO_ERR_PARAM, "peer group: null buffer array");
    if (peer->epoch == 0) return fail(TEMPO_ERR_PARAM, "peer group: epoch starts at 1");
    return TEMPO_OK;
}

static tb::LnPeer to_peer(const tempo_ln_peer_t* p) {
    return tb::LnPeer{p->rank, p->world, p->inbox, p->flags, p->epoch, p->status, p->timeout_ms};
}

int tempo_ln_ip_bwd_peer(const float* dy, const float* y, const float* rstd, const float* gamma,
                         const float* beta, float* dx, float* dgamma, float* dbeta,
                         void* workspace, size_t workspace_bytes, int64_t rows, int64_t cols,
                         const tempo_ln_peer_t* peer, tempo_stream_t stream) {
    if (int rc = check_peer(peer)) return rc;
    if (int rc = check_rows(rows, cols, "layernorm backward")) return rc;
    if (cols > std::numeric_limits<int>::max() / 2)
        return fail(TEMPO_ERR_DIMENSION, "layernorm: row too long");
    if (cols > 0 && (!gamma || !beta || !dgamma || !dbeta))
        return fail(TEMPO_ERR_PARAM, "layernorm: null parameter pointer");
    if (rows > 0 && (!dy || !y || !rstd || !dx))
        return fail(TEMPO_ERR_PARAM, "layernorm: null tensor pointer");
    size_t need = tempo_ln_ip_bwd_workspace_size(rows, cols);
    if (workspace_bytes < need || (need > 0 && !workspace))
        return fail(TEMPO_ERR_PARAM, "layernorm backward workspace too small: need " +
                                         std::to_string(need) + " bytes");
    const tb::LnPeer pg = to_peer(peer);
    return cuda_status(tb::launch_ln_bwd(dy, y, rstd, gamma, beta, dx, dgamma, dbeta, workspace,
                                         rows, cols, S(stream), &pg),
                       "tempo_ln_ip_bwd_peer");
}

int tempo_ln_param_reduce_peer(const double* partials, int64_t nparts, int64_t cols,
                               const tempo_ln_peer_t* peer, float* dgamma, float* dbeta,
                               tempo_stream_t stream) {
    if (int rc = check_peer(peer)) return rc;
    if (nparts < 0 || cols < 0 || cols > std::numeric_limits<int>::max() / 2 ||
        nparts > std::numeric_limits<int>::max())
        return fail(TEMPO_ERR_DIMENSION, "param reduce: bad sizes");
    if (cols > 0 && (!dgamma || !dbeta || (nparts > 0 && !partials)))
        return fail(TEMPO_ERR_PARAM, "param reduce: null pointer");
    return cuda_status(tb::launch_ln_param_reduce_peer(partials, nparts, cols, to_peer(peer),
                                                       dgamma, dbeta, S(stream)),
                       "tempo_ln_param_reduce_peer");
}

// ---- NCCL fallback for the dgamma/dbeta sum -------------------
// libnccl is loaded at first use (dlopen of the soname: inside a PyTorch
// process this resolves to the NCCL torch already loaded), so the library
// itself has no NCCL link dependency and the peer-memory path needs none.
namespace {
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string load_error;
};
const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.load_error = std::string("cannot load libnccl: ") + (e ? e : "?");
            return a;
        }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce ||
            !a.error_string)
            a.load_error = "libnccl lacks an expected symbol";
        return a;
    }();
    return api;
}
int nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return TEMPO_OK;
    return fail(TEMPO_ERR_CUDA, std::string(what) + ": " + nccl().error_string(r));
}
}  // namespace

int tempo_nccl_unique_id(void* id128) {
    if (!id128) return fail(TEMPO_ERR_PARAM, "nccl unique id: null pointer");
    const NcclApi& a = nccl();
    if (!a.load_error.empty()) return fail(TEMPO_ERR_UNSUPPORTED, a.load_error);
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    int rc = nccl_status(a.get_unique_id(&id), "ncclGetUniqueId");
    if (rc == TEMPO_OK) std::memcpy(id128, &id, sizeof(id));
    return rc;
}

int tempo_nccl_comm_init(int32_t world, int32_t rank, const void* id128, void** comm) {
    if (!id128 || !comm) return fail(TEMPO_ERR_PARAM, "nccl comm init: null pointer");
    if (world < 1 || rank < 0 || rank >= world)
        return fail(TEMPO_ERR_PARAM, "nccl comm init: rank " + std::to_string(rank) + " of " +
                                         std::to_string(world));
    const NcclApi& a = nccl();
    if (!a.load_error.empty()) return fail(TEMPO_ERR_UNSUPPORTED, a.load_error);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    int rc = nccl_status(a.comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
    *comm = rc == TEMPO_OK ? static_cast<void*>(c) : nullptr;
    return rc;
}

int tempo_nccl_comm_destroy(void* comm) {
    if (!comm) return TEMPO_OK;
    const NcclApi& a = nccl();
    if (!a.load_error.empty()) return fail(TEMPO_ERR_UNSUPPORTED, a.load_error);
    return nccl_status(a.comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

int tempo_allreduce_ln_params(void* nccl_comm, float* bucket, int64_t count,
                              tempo_stream_t stream) {
    if (count < 0) return fail(TEMPO_ERR_DIMENSION, "allreduce: negative count");
    if (count == 0) return TEMPO_OK;
    if (!nccl_comm || !bucket) return fail(TEMPO_ERR_PARAM, "allreduce: null pointer");
    const NcclApi& a = nccl();
    if (!a.load_error.empty()) return fail(TEMPO_ERR_UNSUPPORTED, a.load_error);
    return nccl_status(a.all_reduce(bucket, bucket, (size_t)count, ncclFloat32, ncclSum,
                                    static_cast<ncclComm_t>(nccl_comm), S(stream)),
                       "ncclAllReduce");
}

int tempo_peer_alloc(size_t bytes, void** dev_ptr) {
    if (!dev_ptr) return fail(TEMPO_ERR_PARAM, "peer alloc: null out pointer");
    *dev_ptr = nullptr;
    cudaError_t e = cudaMalloc(dev_ptr, bytes > 0 ? bytes : 1);
    if (e == cudaSuccess) e = cudaMemset(*dev_ptr, 0, bytes > 0 ? bytes : 1);
    return cuda_status(e, "tempo_peer_alloc");
}

int tempo_peer_free(void* dev_ptr) {
    if (!dev_ptr) return TEMPO_OK;
    return cuda_status(cudaFree(dev_ptr), "tempo_peer_free");
}

int tempo_ipc_get_handle(const void* dev_ptr, void* handle64) {
    if (!dev_ptr || !handle64) return fail(TEMPO_ERR_PARAM, "ipc: null pointer");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
    if (e != cudaSuccess) return cuda_status(e, "tempo_ipc_get_handle");
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
    return TEMPO_OK;
}

int tempo_ipc_open_handle(const void* handle64, void** dev_ptr) {
    if (!handle64 || !dev_ptr) return fail(TEMPO_ERR_PARAM, "ipc: null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    return cuda_status(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess),
                       "tempo_ipc_open_handle");
}

int tempo_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return TEMPO_OK;
    return cuda_status(cudaIpcCloseMemHandle(dev_ptr), "tempo_ipc_close");
}

// ---- softmax / attention dropout -------------------------------------------------
int tempo_softmax_ip_fwd(const float* z, float* P, int64_t rows, int64_t cols,
                         tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "softmax")) return rc;
    return cuda_status(tb::launch_softmax_fwd(z, P, rows, cols, S(stream)), "tempo_softmax_ip_fwd");
}

int tempo_softmax_ip_bwd(const float* dP, const float* P, float* dZ, int64_t rows, int64_t cols,
                         tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "softmax backward")) return rc;
    return cuda_status(tb::launch_softmax_bwd(dP, P, dZ, rows, cols, S(stream)),
                       "tempo_softmax_ip_bwd");
}

int tempo_softmax_dropout_fwd(const float* z, double p, tempo_mask_mode_t mode, uint32_t* mask,
                              uint64_t seed, uint64_t offset, float* P, float* D, int64_t rows,
                              int64_t cols, tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "softmax")) return rc;
    if (int rc = check_p(p)) return rc;
    if (int rc = check_mode(mode)) return rc;
    if (rows > 0 && (!z || !P || !mask)) return fail(TEMPO_ERR_PARAM, "softmax: null pointer");
    return cuda_status(tb::launch_softmax_dropout_fwd(z, 1.0 / (1.0 - p), philox_threshold(p),
                                                      mode == TEMPO_MASK_PHILOX, mask, seed,
                                                      offset, P, D, rows, cols, S(stream)),
                       "tempo_softmax_dropout_fwd");
}

int tempo_attn_probs_bwd(const float* dD, const float* P, const uint32_t* mask, double p,
                         float* dZ, float* D_out, int64_t rows, int64_t cols,
                         tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "softmax backward")) return rc;
    if (int rc = check_p(p)) return rc;
    if (rows > 0 && (!dD || !P || !mask || !dZ))
        return fail(TEMPO_ERR_PARAM, "attn_probs_bwd: null pointer");
    return cuda_status(tb::launch_attn_probs_bwd(dD, P, mask, 1.0 / (1.0 - p), dZ, D_out, rows,
                                                 cols, S(stream)),
                       "tempo_attn_probs_bwd");
}

// ---- dropout -------------------------------------------------------------------
int tempo_attn_dropout_ctx(const float* P, const uint32_t* mask, double p, const float* V,
                           float* ctx, int64_t heads, int64_t s_q, int64_t s_k, int64_t d,
                           tempo_stream_t stream) {
    if (heads < 0 || s_q < 0 || s_k < 0 || d < 0)
        return fail(TEMPO_ERR_DIMENSION, "attn_dropout_ctx: negative shape");
    if (int rc = check_p(p)) return rc;
    if (heads == 0) return TEMPO_OK;
    if (!tb::ctx_gemm_supported(s_q, s_k, d))
        return fail(TEMPO_ERR_UNSUPPORTED,
                    "attn_dropout_ctx needs s_k % 32 == 0 and d in {32, 64}; "
                    "use tempo_softmax_dropout_fwd with D and a GEMM");
    if (!P || !mask || !V || !ctx) return fail(TEMPO_ERR_PARAM, "attn_dropout_ctx: null pointer");
    if (((uintptr_t)P | (uintptr_t)V | (uintptr_t)ctx) & 15u)
        return fail(TEMPO_ERR_ALIGNMENT, "attn_dropout_ctx: P, V and ctx must be 16-byte aligned");
    return cuda_status(tb::launch_ctx_recompute_gemm(P, mask, 1.0 / (1.0 - p), V, ctx, heads, s_q,
                                                     s_k, d, S(stream)),
                       "tempo_attn_dropout_ctx");
}

int tempo_attn_dropout_dv(const float* P, const uint32_t* mask, double p, const float* dO,
                          float* dV, int64_t heads, int64_t s_q, int64_t s_k, int64_t d,
                          tempo_stream_t stream) {
    if (heads < 0 || s_q < 0 || s_k < 0 || d < 0)
        return fail(TEMPO_ERR_DIMENSION, "attn_dropout_dv: negative shape");
    if (int rc = check_p(p)) return rc;
    if (heads == 0) return TEMPO_OK;
    if (!tb::dv_gemm_supported(s_q, s_k, d))
        return fail(TEMPO_ERR_UNSUPPORTED,
                    "attn_dropout_dv needs s_q % 32 == 0, s_k % 256 == 0 and d in {32, 64, 128}; "
                    "use tempo_attn_probs_bwd with D_out and a GEMM");
    if (!P || !mask || !dO || !dV) return fail(TEMPO_ERR_PARAM, "attn_dropout_dv: null pointer");
    if (((uintptr_t)P | (uintptr_t)dO | (uintptr_t)dV) & 15u)
        return fail(TEMPO_ERR_ALIGNMENT, "attn_dropout_dv: P, dO and dV must be 16-byte aligned");
    return cuda_status(tb::launch_dv_recompute_gemm(P, mask, 1.0 / (1.0 - p), dO, dV, heads, s_q,
                                                    s_k, d, S(stream)),
                       "tempo_attn_dropout_dv");
}

int tempo_dropout_add_ln_fwd(const float* proj, const float* residual, double p,
                             tempo_mask_mode_t mode, uint32_t* mask, uint64_t seed,
                             uint64_t offset, const float* gamma, const float* beta, double eps,
                             float* y, float* rstd, int64_t rows, int64_t cols,
                             int32_t* dev_status, tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "dropout_add_layernorm")) return rc;
    if (int rc = check_p(p)) return rc;
    if (int rc = check_mode(mode)) return rc;
    if (!(eps > 0.0)) return fail(TEMPO_ERR_PARAM, "layernorm epsilon must be positive");
    if (cols % 32 != 0)
        return fail(TEMPO_ERR_UNSUPPORTED,
                    "dropout_add_layernorm needs cols % 32 == 0 (rows own whole mask words); "
                    "use tempo_dropout_fwd + add + tempo_ln_ip_fwd");
    if (cols > (1 << 14)) return fail(TEMPO_ERR_DIMENSION, "dropout_add_layernorm: row too long");
    if (rows > 0 && (!proj || !residual || !mask || !gamma || !beta || !y || !rstd))
        return fail(TEMPO_ERR_PARAM, "dropout_add_layernorm: null pointer");
    return cuda_status(tb::launch_dal_fwd(proj, residual, 1.0 / (1.0 - p), philox_threshold(p),
                                          mode == TEMPO_MASK_PHILOX, mask, seed, offset, gamma,
                                          beta, eps, y, rstd, rows, cols, dev_status, S(stream)),
                       "tempo_dropout_add_ln_fwd");
}

int tempo_dropout_add_ln_bwd(const float* dy, const float* y, const float* rstd,
                             const float* gamma, const float* beta, const uint32_t* mask,
                             double p, float* d_residual, float* d_proj, float* dgamma,
                             float* dbeta, void* workspace, size_t workspace_bytes, int64_t rows,
                             int64_t cols, const tempo_ln_peer_t* peer, tempo_stream_t stream) {
    if (peer)
        if (int rc = check_peer(peer)) return rc;
    if (int rc = check_rows(rows, cols, "dropout_add_layernorm backward")) return rc;
    if (int rc = check_p(p)) return rc;
    if (cols > std::numeric_limits<int>::max() / 2)
        return fail(TEMPO_ERR_DIMENSION, "layernorm: row too long");
    if (cols % 4 != 0)
        return fail(TEMPO_ERR_UNSUPPORTED, "dropout_add_layernorm backward needs cols % 4 == 0");
    if (cols > 0 && (!gamma || !beta || !dgamma || !dbeta))
        return fail(TEMPO_ERR_PARAM, "layernorm: null parameter pointer");
    if (rows > 0 && (!dy || !y || !rstd || !d_residual || !d_proj || !mask))
        return fail(TEMPO_ERR_PARAM, "dropout_add_layernorm backward: null tensor pointer");
    size_t need = tempo_ln_ip_bwd_workspace_size(rows, cols);
    if (workspace_bytes < need || (need > 0 && !workspace))
        return fail(TEMPO_ERR_PARAM, "layernorm backward workspace too small: need " +
                                         std::to_string(need) + " bytes");
    tb::LnPeer pg{};
    if (peer) pg = to_peer(peer);
    return cuda_status(tb::launch_ln_bwd(dy, y, rstd, gamma, beta, d_residual, dgamma, dbeta,
                                         workspace, rows, cols, S(stream), peer ? &pg : nullptr,
                                         mask, 1.0 / (1.0 - p), d_proj),
                       "tempo_dropout_add_ln_bwd");
}

int tempo_dropout_fwd(const float* x, double p, tempo_mask_mode_t mode, uint32_t* mask,
                      uint64_t seed, uint64_t offset, float* y, int64_t n, tempo_stream_t stream) {
    if (int rc = check_n(n, "dropout")) return rc;
    if (int rc = check_p(p)) return rc;
    if (int rc = check_mode(mode)) return rc;
    if (n > 0 && (!x || !y || !mask)) return fail(TEMPO_ERR_PARAM, "dropout: null pointer");
    return cuda_status(tb::launch_dropout_fwd(x, 1.0 / (1.0 - p), philox_threshold(p),
                                              mode == TEMPO_MASK_PHILOX, mask, seed, offset, y, n,
                                              S(stream)),
                       "tempo_dropout_fwd");
}

int tempo_dropout_recompute(const float* P, const uint32_t* mask, double p, float* D, int64_t n,
                            tempo_stream_t stream) {
    if (int rc = check_n(n, "dropout recompute")) return rc;
    if (int rc = check_p(p)) return rc;
    if (n > 0 && (!P || !D || !mask)) return fail(TEMPO_ERR_PARAM, "dropout recompute: null pointer");
    return cuda_status(tb::launch_dropout_fwd(P, 1.0 / (1.0 - p), philox_threshold(p), 0,
                                              const_cast<uint32_t*>(mask), 0, 0, D, n, S(stream)),
                       "tempo_dropout_recompute");
}

int tempo_dropout_bwd(const float* dy, const uint32_t* mask, double p, float* dx, int64_t n,
                      tempo_stream_t stream) {
    if (int rc = check_n(n, "dropout")) return rc;
    if (int rc = check_p(p)) return rc;
    if (n > 0 && (!dy || !dx || !mask)) return fail(TEMPO_ERR_PARAM, "dropout: null pointer");
    return cuda_status(tb::launch_dropout_bwd(dy, mask, 1.0 / (1.0 - p), dx, n, S(stream)),
                       "tempo_dropout_bwd");
}

int tempo_tensor_scale(const float* a, double c, float* out, int64_t n, tempo_stream_t stream) {
    if (int rc = check_n(n, "tensor")) return rc;
    return cuda_status(tb::launch_scale(a, c, out, n, S(stream)), "tempo_tensor_scale");
}

int tempo_tensor_add(const float* a, const float* b, float* out, int64_t n,
                     tempo_stream_t stream) {
    if (int rc = check_n(n, "add")) return rc;
    if (n > 0 && (!a || !b || !out)) return fail(TEMPO_ERR_PARAM, "add: null pointer");
    return cuda_status(tb::launch_add(a, b, out, n, S(stream)), "tempo_tensor_add");
}

// ---- masks ---------------------------------------------------------------------
int tempo_mask_pack(const uint8_t* bytes, uint32_t* bits, int64_t n, int32_t* dev_status,
                    tempo_stream_t stream) {
    if (int rc = check_n(n, "mask")) return rc;
    return cuda_status(tb::launch_mask_pack(bytes, bits, n, dev_status, S(stream)),
                       "tempo_mask_pack");
}

int tempo_mask_unpack(const uint32_t* bits, uint8_t* bytes, int64_t n, tempo_stream_t stream) {
    if (int rc = check_n(n, "mask")) return rc;
    return cuda_status(tb::launch_mask_unpack(bits, bytes, n, S(stream)), "tempo_mask_unpack");
}

int tempo_bernoulli_keep_bits_host(int64_t n, double p, uint64_t seed, uint32_t* bits) {
    if (int rc = check_n(n, "mask")) return rc;
    if (!(p >= 0.0) || p >= 1.0)  // tensor.cpp:188-191
        return fail(TEMPO_ERR_PARAM,
                    "drop probability must lie in [0, 1), got " + std::to_string(p));
    // tensor.cpp:197-201: one std::mt19937_64 stream, uniform_real_distribution
    // <double>(0, 1), keep <=> u >= p, element order.
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(0.0, 1.0);
    const int64_t words = (n + 31) / 32;
    for (int64_t w = 0; w < words; ++w) {
        uint32_t word = 0;
        const int64_t lim = std::min<int64_t>(32, n - w * 32);
        for (int64_t b = 0; b < lim; ++b)
            if (dist(rng) >= p) word |= 1u << b;
        bits[w] = word;
    }
    return TEMPO_OK;
}

size_t tempo_bernoulli_keep_bits_workspace_size(uint64_t offset, int64_t n) {
    return n > 0 ? tb::mt_keep_workspace(offset, n) : 0;
}

int tempo_bernoulli_keep_bits(int64_t n, double p, uint64_t seed, uint64_t offset,
                              uint32_t* bits, void* workspace, size_t workspace_bytes,
                              tempo_stream_t stream) {
    if (int rc = check_n(n, "mask")) return rc;
    if (!(p >= 0.0) || p >= 1.0)  // tensor.cpp:188-191
        return fail(TEMPO_ERR_PARAM,
                    "drop probability must lie in [0, 1), got " + std::to_string(p));
    if (offset % 32 != 0)
        return fail(TEMPO_ERR_PARAM, "offset must be a multiple of 32 (whole mask words)");
    if (n == 0) return TEMPO_OK;
    if (!bits) return fail(TEMPO_ERR_PARAM, "null mask");
    const size_t need = tb::mt_keep_workspace(offset, n);
    if (workspace_bytes < need || (need && !workspace))
        return fail(TEMPO_ERR_PARAM, "workspace too small: need " + std::to_string(need) +
                                         " bytes");
    return cuda_status(tb::launch_mt_keep_bits(seed, p, offset, n, bits, workspace,
                                               workspace_bytes, S(stream)),
                       "tempo_bernoulli_keep_bits");
}

int tempo_softmax_dropout_fwd_refmask(const float* z, double p, uint64_t seed, uint64_t offset,
                                      uint32_t* mask, float* P, float* D, int64_t rows,
                                      int64_t cols, void* workspace, size_t workspace_bytes,
                                      tempo_stream_t stream) {
    if (int rc = check_rows(rows, cols, "softmax")) return rc;
    if (int rc = check_p(p)) return rc;
    if (offset % 32 != 0)
        return fail(TEMPO_ERR_PARAM, "offset must be a multiple of 32 (whole mask words)");
    if (rows == 0 || cols == 0) return TEMPO_OK;
    if (!z || !P || !mask) return fail(TEMPO_ERR_PARAM, "softmax: null pointer");
    const size_t need = tb::mt_keep_workspace(offset, rows * cols);
    if (workspace_bytes < need || (need && !workspace))
        return fail(TEMPO_ERR_PARAM, "workspace too small: need " + std::to_string(need) +
                                         " bytes");
    return cuda_status(tb::launch_softmax_dropout_fwd_mt(z, p, seed, offset, mask, P, D, rows,
                                                         cols, workspace, workspace_bytes,
                                                         S(stream)),
                       "tempo_softmax_dropout_fwd_refmask");
}

uint64_t tempo_mask_stream_seed(uint64_t mask_seed, uint64_t salt, int site) {
    // encoder.cpp:39-46 (splitmix64 over a site-salted input)
    uint64_t z = mask_seed + 0x9E3779B97F4A7C15ull * (salt * 3 + (uint64_t)site + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---- stash accounting ------------------------------------------------------------
int64_t tempo_layer_stash_bytes_per_token(int64_t seq, int64_t hidden, int64_t heads,
                                          int tempo_variant, int mask_bits) {
    // memory_model.cpp:31-65 inventory at fp32 + masks; Tempo removes the
    // GELU input (16H, adds a 4H mask), both LN inputs (8H, adds 2 rstd
    // floats), the dropped-out map (4AS) and the softmax input (4AS).
    const int64_t H = hidden, AS = heads * seq;
    int64_t float_bytes, mask_elems;
    if (tempo_variant) {
        float_bytes = 4 * (H + 3 * H + AS + H + H + 4 * H) + 8;  // input,qkv,P,ctx,ln1_out,gelu_out
        mask_elems = AS + H + 4 * H + H;  // attn drop, attn-out drop, gelu branch, ffn drop
    } else {
        float_bytes = 4 * (H + 3 * H + 3 * AS + H + H + H + 4 * H + 4 * H + H);
        mask_elems = AS + H + H;
    }
    int64_t mask_bytes_x8 = mask_bits ? mask_elems : 8 * mask_elems;
    return float_bytes + mask_bytes_x8 / 8;
}

}  // extern "C"
