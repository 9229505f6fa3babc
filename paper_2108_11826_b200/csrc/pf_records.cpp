// pf_records.cpp — poses.jsonl lines for a whole batch (operators.py:293-310
// pose_record), byte-identical to the reference's
//   json.dumps({"frame_id": seq, "humans": [{"score": s, "keypoints":
//       [{"part": name, "x": x, "y": y, "score": ks}, ...]}, ...]},
//       separators=(",", ":"))
// Floats are printed as CPython's repr: the shortest digit string that
// round-trips (std::to_chars gives the same digits), fixed notation for
// decimal-point positions in (-4, 16], else d.ddde±XX (at least two exponent
// digits); "Infinity" / "NaN" as json.dumps writes them.  SURVEY.md §8(f) 3.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/pf_b200.h"

namespace {

void put_float(std::string &o, double v)
{
    if (std::isnan(v)) { o += "NaN"; return; }
    if (std::isinf(v)) { o += v > 0 ? "Infinity" : "-Infinity"; return; }
    if (v == 0.0) { o += std::signbit(v) ? "-0.0" : "0.0"; return; }
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    // buf = [-]d[.ddd]e(+|-)XX
    const char *p = buf, *end = r.ptr;
    bool neg = false;
    if (*p == '-') { neg = true; ++p; }
    char digits[32];
    int nd = 0;
    const char *e = p;
    while (e < end && *e != 'e') {
        if (*e != '.') digits[nd++] = *e;
        ++e;
    }
    int exp10 = 0;                           // value = d.ddd x 10^exp10 (buf is not NUL-terminated)
    {
        const char *q = e + 1;
        const bool eneg = q < end && *q == '-';
        if (q < end && (*q == '-' || *q == '+')) ++q;
        for (; q < end; ++q) exp10 = exp10 * 10 + (*q - '0');
        if (eneg) exp10 = -exp10;
    }
    const int decpt = exp10 + 1;             // value = 0.ddd x 10^decpt (CPython's decpt)
    if (neg) o += '-';
    if (decpt <= -4 || decpt > 16) {
        o += digits[0];
        if (nd > 1) { o += '.'; o.append(digits + 1, nd - 1); }
        o += 'e';
        const int x = decpt - 1;
        o += x < 0 ? '-' : '+';
        const int ax = x < 0 ? -x : x;
        if (ax < 10) o += '0';
        o += std::to_string(ax);
    } else if (decpt <= 0) {
        o += "0.";
        o.append(-decpt, '0');
        o.append(digits, nd);
    } else if (decpt >= nd) {
        o.append(digits, nd);
        o.append(decpt - nd, '0');
        o += ".0";
    } else {
        o.append(digits, decpt);
        o += '.';
        o.append(digits + decpt, nd - decpt);
    }
}

// json.dumps string escaping (ensure_ascii=True) for the part names: the
// UTF-8 bytes are decoded to code points; every one outside ' '..'~' becomes
// \uXXXX, with a surrogate pair above U+FFFF (CPython's py_encode_basestring_ascii).
void put_u16(std::string &o, unsigned v)
{
    char u[8];
    std::snprintf(u, sizeof(u), "\\u%04x", v);
    o += u;
}

void put_string(std::string &o, const char *s)
{
    o += '"';
    const unsigned char *c = reinterpret_cast<const unsigned char *>(s);
    while (*c) {
        unsigned cp = *c++;
        if (cp >= 0x80) {   // multi-byte sequence (names come from Python str.encode(): valid UTF-8)
            const int extra = cp >= 0xf0 ? 3 : cp >= 0xe0 ? 2 : 1;
            cp &= extra == 3 ? 0x07u : extra == 2 ? 0x0fu : 0x1fu;
            for (int k = 0; k < extra && (*c & 0xc0) == 0x80; ++k) cp = (cp << 6) | (*c++ & 0x3fu);
        }
        switch (cp) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        default:
            if (cp < 0x20 || cp >= 0x7f) {
                if (cp > 0xffff) {
                    cp -= 0x10000;
                    put_u16(o, 0xd800 | (cp >> 10));
                    put_u16(o, 0xdc00 | (cp & 0x3ff));
                } else {
                    put_u16(o, cp);
                }
            } else {
                o += static_cast<char>(cp);
            }
        }
    }
    o += '"';
}

}  // namespace

extern "C" {

long long pf_format_records(int n_frames, int n_keypoints, const int32_t *frame_first, const int32_t *frame_count,
                            const double *human_score, const double *kp_x, const double *kp_y,
                            const float *kp_score, const int32_t *kp_peak, const char *const *part_names,
                            long long seq_base, char *out, long long cap)
{
    if (n_frames < 0 || n_keypoints < 0 || (n_frames > 0 && (!frame_first || !frame_count))) return -1;
    std::string o;
    o.reserve((size_t)n_frames * 64);
    for (int f = 0; f < n_frames; ++f) {
        o += "{\"frame_id\":";
        o += std::to_string(seq_base + f);
        o += ",\"humans\":[";
        for (int h = frame_first[f], hn = 0; hn < frame_count[f]; ++h, ++hn) {
            if (hn) o += ',';
            o += "{\"score\":";
            put_float(o, human_score[h]);
            o += ",\"keypoints\":[";
            bool first = true;
            for (int k = 0; k < n_keypoints; ++k) {
                const size_t i = (size_t)h * n_keypoints + k;
                if (kp_peak[i] < 0) continue;
                if (!first) o += ',';
                first = false;
                o += "{\"part\":";
                put_string(o, part_names[k]);
                o += ",\"x\":";
                put_float(o, kp_x[i]);
                o += ",\"y\":";
                put_float(o, kp_y[i]);
                o += ",\"score\":";
                put_float(o, (double)kp_score[i]);
                o += '}';
            }
            o += "]}";
        }
        o += "]}\n";
    }
    const long long n = (long long)o.size();
    if (out && cap >= n) std::memcpy(out, o.data(), (size_t)n);
    return n;
}

// One float as CPython repr (for the formatter's tests).
int pf_format_float(double v, char *out, int cap)
{
    std::string o;
    put_float(o, v);
    if ((int)o.size() + 1 > cap) return -1;
    std::memcpy(out, o.c_str(), o.size() + 1);
    return (int)o.size();
}

}  // extern "C"
