// merf_bundle.cu -- NEXT-4 asset ingestion: the on-disk bundle of a baked scene and camera
// files (Sec. 5.3 P:274-276 "we encode textures as PNGs"; SPEC S:430-465 layout).
// Host code only (zlib for the PNG streams); the scene is then uploaded with
// merf_scene_upload.  Layout of a bundle directory (version 1):
//   manifest.txt                 key/value lines, MLP weights in decimal (%.9g: exact fp32),
//                                one "file <name> <bytes> <crc32>" line per payload
//   plane<a>_{density,diffuse,features}.png   a = 0..2: 8-bit gray / RGB / RGBA, R x R
//   atlas_{density,diffuse,features}.png      Z-major stack of 9x9 block slices (slice
//                                q = 9 b + z), 455 slices per raster row (<= 4095 px wide)
//   block_index.bin              int32 little-endian [(L/8)^3], -1 = empty
//   occupancy<i>.bin             level i (coarse -> fine): bit k of byte n = cell 8n + k,
//                                x fastest, ceil(N^3 / 8) bytes
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <sys/stat.h>
#include <zlib.h>

#include "../../include/merf.h"

merf_status merf_set_error(merf_status s, const char* msg);   // merf_api.cu

namespace {

merf_status efail(merf_status s, const char* fmt, ...) {
    char buf[640];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    return merf_set_error(s, buf);
}

constexpr int kVersion = 1;
constexpr int kSlicesPerRow = 455;   // 455 * 9 = 4095 <= 4096 px

// ------------------------------------------------------------------------------------
// PNG (8-bit gray / RGB / RGBA, no interlace)
// ------------------------------------------------------------------------------------
void put_be32(std::vector<uint8_t>& v, uint32_t x) {
    v.push_back(uint8_t(x >> 24));
    v.push_back(uint8_t(x >> 16));
    v.push_back(uint8_t(x >> 8));
    v.push_back(uint8_t(x));
}
uint32_t get_be32(const uint8_t* p) { return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3]; }

void put_chunk(std::vector<uint8_t>& out, const char* type, const uint8_t* data, size_t n) {
    put_be32(out, (uint32_t)n);
    const size_t at = out.size();
    out.insert(out.end(), type, type + 4);
    if (n) out.insert(out.end(), data, data + n);
    const uint32_t crc = (uint32_t)crc32_z(0L, out.data() + at, n + 4);
    put_be32(out, crc);
}

int color_type(int ch) { return ch == 1 ? 0 : ch == 3 ? 2 : 6; }

// pixels [h][w][ch] -> PNG bytes (filter type 0 on every row)
bool png_encode(const uint8_t* px, int w, int h, int ch, std::vector<uint8_t>& out) {
    const size_t row = (size_t)w * ch;
    std::vector<uint8_t> raw((row + 1) * h);
    for (int y = 0; y < h; y++) {
        raw[y * (row + 1)] = 0;
        memcpy(&raw[y * (row + 1) + 1], px + y * row, row);
    }
    uLongf zn = compressBound((uLong)raw.size());
    std::vector<uint8_t> z(zn);
    if (compress2(z.data(), &zn, raw.data(), (uLong)raw.size(), 6) != Z_OK) return false;
    static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    out.assign(sig, sig + 8);
    std::vector<uint8_t> ihdr;
    put_be32(ihdr, (uint32_t)w);
    put_be32(ihdr, (uint32_t)h);
    ihdr.push_back(8);
    ihdr.push_back((uint8_t)color_type(ch));
    ihdr.push_back(0);
    ihdr.push_back(0);
    ihdr.push_back(0);
    put_chunk(out, "IHDR", ihdr.data(), ihdr.size());
    const size_t kIdat = size_t(1) << 24;
    for (size_t o = 0; o < zn; o += kIdat) put_chunk(out, "IDAT", z.data() + o, std::min(kIdat, (size_t)zn - o));
    put_chunk(out, "IEND", nullptr, 0);
    return true;
}

uint8_t paeth(int a, int b, int c) {
    const int p = a + b - c, pa = abs(p - a), pb = abs(p - b), pc = abs(p - c);
    return (uint8_t)((pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c));
}

// PNG bytes -> pixels [h][w][ch]; the expected shape must match exactly
merf_status png_decode(const std::vector<uint8_t>& f, const char* name, int w, int h, int ch, uint8_t* px) {
    static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    if (f.size() < 8 || memcmp(f.data(), sig, 8) != 0) return efail(MERF_EIO, "%s: not a PNG file", name);
    size_t p = 8;
    std::vector<uint8_t> z;
    bool hdr = false, end = false;
    while (p + 12 <= f.size() && !end) {
        const uint32_t n = get_be32(&f[p]);
        if (p + 12 + (size_t)n > f.size()) return efail(MERF_EIO, "%s: truncated chunk", name);
        const uint8_t* type = &f[p + 4];
        const uint8_t* data = &f[p + 8];
        if ((uint32_t)crc32_z(0L, type, (size_t)n + 4) != get_be32(&f[p + 8 + n]))
            return efail(MERF_EIO, "%s: chunk CRC mismatch", name);
        if (!memcmp(type, "IHDR", 4)) {
            if (n != 13) return efail(MERF_EIO, "%s: bad IHDR", name);
            const int gw = (int)get_be32(data), gh = (int)get_be32(data + 4);
            if (data[8] != 8 || data[9] != color_type(ch) || data[10] || data[11] || data[12])
                return efail(MERF_EIO, "%s: expected 8-bit non-interlaced colour type %d", name, color_type(ch));
            if (gw != w || gh != h)
                return efail(MERF_EIO, "%s: size mismatch: %dx%d in file, %dx%d from the manifest", name, gw, gh, w, h);
            hdr = true;
        } else if (!memcmp(type, "IDAT", 4)) {
            z.insert(z.end(), data, data + n);
        } else if (!memcmp(type, "IEND", 4)) {
            end = true;
        }
        p += 12 + n;
    }
    if (!hdr || !end) return efail(MERF_EIO, "%s: missing IHDR or IEND", name);
    const size_t row = (size_t)w * ch;
    std::vector<uint8_t> raw((row + 1) * h);
    uLongf rn = (uLongf)raw.size();
    if (uncompress(raw.data(), &rn, z.data(), (uLong)z.size()) != Z_OK || rn != raw.size())
        return efail(MERF_EIO, "%s: corrupt image data", name);
    for (int y = 0; y < h; y++) {
        const uint8_t ft = raw[y * (row + 1)];
        const uint8_t* src = &raw[y * (row + 1) + 1];
        uint8_t* dst = px + y * row;
        const uint8_t* up = y ? px + (y - 1) * row : nullptr;
        for (size_t i = 0; i < row; i++) {
            const int a = i >= (size_t)ch ? dst[i - ch] : 0;
            const int b = up ? up[i] : 0;
            const int c = (up && i >= (size_t)ch) ? up[i - ch] : 0;
            int v = src[i];
            switch (ft) {
                case 0: break;
                case 1: v += a; break;
                case 2: v += b; break;
                case 3: v += (a + b) >> 1; break;
                case 4: v += paeth(a, b, c); break;
                default: return efail(MERF_EIO, "%s: bad filter type %d", name, ft);
            }
            dst[i] = (uint8_t)v;
        }
    }
    return MERF_OK;
}

// ------------------------------------------------------------------------------------
// files
// ------------------------------------------------------------------------------------
std::string join(const char* dir, const std::string& name) { return std::string(dir) + "/" + name; }

bool write_file(const std::string& path, const void* p, size_t n) {
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) return false;
    const bool ok = fwrite(p, 1, n, f) == n;
    return fclose(f) == 0 && ok;
}

bool read_file(const std::string& path, std::vector<uint8_t>& out) {
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    const long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    out.resize(n > 0 ? (size_t)n : 0);
    const bool ok = n >= 0 && fread(out.data(), 1, out.size(), f) == out.size();
    fclose(f);
    return ok;
}

struct Payload {
    std::string name;
    std::vector<uint8_t> bytes;
};

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int64_t occ_bytes(int N) { return ((int64_t)N * N * N + 7) / 8; }

// OR-pool the finest bits into level `Nc` (x fastest, LSB first)
std::vector<uint8_t> pool_bits(const uint8_t* fine, int N, int Nc) {
    std::vector<uint8_t> out(occ_bytes(Nc), 0);
    const int f = N / Nc;
    for (int64_t z = 0; z < N; z++)
        for (int64_t y = 0; y < N; y++)
            for (int64_t x = 0; x < N; x++) {
                const int64_t i = (z * N + y) * N + x;
                if ((fine[i >> 3] >> (i & 7)) & 1) {
                    const int64_t j = ((z / f) * Nc + y / f) * Nc + x / f;
                    out[j >> 3] |= uint8_t(1u << (j & 7));
                }
            }
    return out;
}

// split [n][C=8] bytes into density (1), diffuse (3), features (4) channel planes
void split_channels(const uint8_t* src, int64_t n, uint8_t* d, uint8_t* rgb, uint8_t* feat) {
    for (int64_t i = 0; i < n; i++) {
        d[i] = src[i * 8];
        for (int c = 0; c < 3; c++) rgb[i * 3 + c] = src[i * 8 + 1 + c];
        for (int c = 0; c < 4; c++) feat[i * 4 + c] = src[i * 8 + 4 + c];
    }
}

void atlas_raster_dims(int64_t n_blocks, int& w, int& h) {
    const int64_t slices = n_blocks * 9;
    const int64_t per_row = slices < kSlicesPerRow ? slices : kSlicesPerRow;
    w = (int)(per_row * 9);
    h = (int)(((slices + kSlicesPerRow - 1) / kSlicesPerRow) * 9);
}

// atlas [n][9][9][9][8] <-> 8-channel raster [h][w][8] of 9x9 slices q = 9 b + z
void atlas_to_raster(const uint8_t* atlas, int64_t n_blocks, int w, uint8_t* ras) {
    for (int64_t q = 0; q < n_blocks * 9; q++) {
        const int64_t X0 = (q % kSlicesPerRow) * 9, Y0 = (q / kSlicesPerRow) * 9;
        for (int y = 0; y < 9; y++)
            memcpy(ras + ((Y0 + y) * w + X0) * 8, atlas + (q * 81 + y * 9) * 8, 9 * 8);
    }
}
void raster_to_atlas(const uint8_t* ras, int64_t n_blocks, int w, uint8_t* atlas) {
    for (int64_t q = 0; q < n_blocks * 9; q++) {
        const int64_t X0 = (q % kSlicesPerRow) * 9, Y0 = (q / kSlicesPerRow) * 9;
        for (int y = 0; y < 9; y++)
            memcpy(atlas + (q * 81 + y * 9) * 8, ras + ((Y0 + y) * w + X0) * 8, 9 * 8);
    }
}

merf_status check_desc(const merf_scene_desc* d) {
    if (d->C != 8) return efail(MERF_EINVAL, "C must be 8");
    if (d->L != 0 && (!is_pow2(d->L) || d->L < 8)) return efail(MERF_EINVAL, "L must be 0 or a power of two >= 8");
    if (d->R != 0 && !is_pow2(d->R)) return efail(MERF_EINVAL, "R must be 0 or a power of two");
    if (d->n_levels < 1 || d->n_levels > MERF_MAX_LEVELS) return efail(MERF_EINVAL, "bad n_levels");
    for (int i = 0; i < d->n_levels; i++) {
        if (!is_pow2(d->level_res[i]) || d->level_res[i] > 4096) return efail(MERF_EINVAL, "bad level_res");
        if (i && d->level_res[i] % d->level_res[i - 1]) return efail(MERF_EINVAL, "levels must divide");
    }
    return MERF_OK;
}

// the 8-channel payload of one image as three PNGs
bool encode_split(const uint8_t* src8, int w, int h, const std::string& stem, std::vector<Payload>& out) {
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> d(n), rgb(n * 3), feat(n * 4);
    split_channels(src8, n, d.data(), rgb.data(), feat.data());
    Payload a{stem + "_density.png", {}}, b{stem + "_diffuse.png", {}}, c{stem + "_features.png", {}};
    if (!png_encode(d.data(), w, h, 1, a.bytes) || !png_encode(rgb.data(), w, h, 3, b.bytes) ||
        !png_encode(feat.data(), w, h, 4, c.bytes))
        return false;
    out.push_back(std::move(a));
    out.push_back(std::move(b));
    out.push_back(std::move(c));
    return true;
}

// ------------------------------------------------------------------------------------
// manifest
// ------------------------------------------------------------------------------------
struct Manifest {
    merf_scene_desc desc{};
    int64_t n_blocks = 0;
    std::vector<float> mlp;
    struct F {
        std::string name;
        uint64_t bytes;
        uint32_t crc;
    };
    std::vector<F> files;
};

merf_status parse_manifest(const char* dir, Manifest& m) {
    std::vector<uint8_t> txt;
    if (!read_file(join(dir, "manifest.txt"), txt)) return efail(MERF_EIO, "%s/manifest.txt: cannot read", dir);
    txt.push_back(0);
    char* save = nullptr;
    int line_no = 0, version = -1;
    bool have_mlp = false;
    for (char* line = strtok_r((char*)txt.data(), "\n", &save); line; line = strtok_r(nullptr, "\n", &save)) {
        line_no++;
        char key[64] = {0};
        int off = 0;
        if (line[0] == '#' || sscanf(line, "%63s%n", key, &off) != 1) continue;
        const char* rest = line + off;
        auto bad = [&](const char* what) { return efail(MERF_EIO, "manifest.txt line %d: bad %s", line_no, what); };
        if (!strcmp(key, "merf_bundle")) {
            if (sscanf(rest, "%d", &version) != 1) return bad("version");
        } else if (!strcmp(key, "L")) {
            if (sscanf(rest, "%d", &m.desc.L) != 1) return bad("L");
        } else if (!strcmp(key, "R")) {
            if (sscanf(rest, "%d", &m.desc.R) != 1) return bad("R");
        } else if (!strcmp(key, "C")) {
            if (sscanf(rest, "%d", &m.desc.C) != 1) return bad("C");
        } else if (!strcmp(key, "block_size")) {
            int b = 0;
            if (sscanf(rest, "%d", &b) != 1 || b != 8) return bad("block_size (must be 8)");
        } else if (!strcmp(key, "level_res")) {
            int n = 0, v, k;
            const char* q = rest;
            while (sscanf(q, "%d%n", &v, &k) == 1 && n < MERF_MAX_LEVELS) {
                m.desc.level_res[n++] = v;
                q += k;
            }
            m.desc.n_levels = n;
        } else if (!strcmp(key, "m_density")) {
            if (sscanf(rest, "%f", &m.desc.m_density) != 1) return bad("m_density");
        } else if (!strcmp(key, "m_appearance")) {
            if (sscanf(rest, "%f", &m.desc.m_appearance) != 1) return bad("m_appearance");
        } else if (!strcmp(key, "step")) {
            if (sscanf(rest, "%lf", &m.desc.step) != 1) return bad("step");
        } else if (!strcmp(key, "t_min")) {
            if (sscanf(rest, "%f", &m.desc.t_min) != 1) return bad("t_min");
        } else if (!strcmp(key, "alpha_skip")) {
            if (sscanf(rest, "%f", &m.desc.alpha_skip) != 1) return bad("alpha_skip");
        } else if (!strcmp(key, "source_mask")) {
            if (sscanf(rest, "%u", &m.desc.source_mask) != 1) return bad("source_mask");
        } else if (!strcmp(key, "n_blocks")) {
            long long nb;
            if (sscanf(rest, "%lld", &nb) != 1 || nb < 0) return bad("n_blocks");
            m.n_blocks = nb;
        } else if (!strcmp(key, "mlp_dims")) {
            int a, b, c, d;
            if (sscanf(rest, "%d %d %d %d", &a, &b, &c, &d) != 4 || a != 34 || b != 16 || c != 16 || d != 3)
                return bad("mlp_dims (must be 34 16 16 3)");
        } else if (!strcmp(key, "mlp")) {
            const char* q = rest;
            float v;
            int k;
            m.mlp.clear();
            while (sscanf(q, "%f%n", &v, &k) == 1) {
                m.mlp.push_back(v);
                q += k;
            }
            if (m.mlp.size() != 883) return bad("mlp (need 883 weights)");
            have_mlp = true;
        } else if (!strcmp(key, "file")) {
            char name[256];
            unsigned long long bytes;
            unsigned crc;
            if (sscanf(rest, "%255s %llu %x", name, &bytes, &crc) != 3) return bad("file entry");
            m.files.push_back({name, bytes, crc});
        }
    }
    if (version < 0) return efail(MERF_EIO, "manifest.txt: missing 'merf_bundle <version>'");
    if (version != kVersion) return efail(MERF_EIO, "bundle version %d, this library reads %d", version, kVersion);
    if (!have_mlp) return efail(MERF_EIO, "manifest.txt: missing mlp weights");
    return check_desc(&m.desc);
}

// read a manifest-listed payload, verifying its size and CRC-32
merf_status load_payload(const char* dir, const Manifest& m, const std::string& name, std::vector<uint8_t>& out) {
    for (auto& f : m.files) {
        if (f.name != name) continue;
        if (!read_file(join(dir, name), out)) return efail(MERF_EIO, "%s: missing payload file", name.c_str());
        if (out.size() != f.bytes) return efail(MERF_EIO, "%s: %zu bytes, manifest says %llu", name.c_str(), out.size(),
                                                (unsigned long long)f.bytes);
        if ((uint32_t)crc32_z(0L, out.data(), out.size()) != f.crc)
            return efail(MERF_EIO, "%s: checksum mismatch", name.c_str());
        return MERF_OK;
    }
    return efail(MERF_EIO, "%s: not listed in the manifest", name.c_str());
}

merf_status decode_split(const char* dir, const Manifest& m, const std::string& stem, int w, int h, uint8_t* dst8) {
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> f, d(n), rgb(n * 3), feat(n * 4);
    merf_status e;
    if ((e = load_payload(dir, m, stem + "_density.png", f)) || (e = png_decode(f, (stem + "_density.png").c_str(), w, h, 1, d.data())))
        return e;
    if ((e = load_payload(dir, m, stem + "_diffuse.png", f)) || (e = png_decode(f, (stem + "_diffuse.png").c_str(), w, h, 3, rgb.data())))
        return e;
    if ((e = load_payload(dir, m, stem + "_features.png", f)) || (e = png_decode(f, (stem + "_features.png").c_str(), w, h, 4, feat.data())))
        return e;
    for (int64_t i = 0; i < n; i++) {
        dst8[i * 8] = d[i];
        for (int c = 0; c < 3; c++) dst8[i * 8 + 1 + c] = rgb[i * 3 + c];
        for (int c = 0; c < 4; c++) dst8[i * 8 + 4 + c] = feat[i * 4 + c];
    }
    return MERF_OK;
}

}  // namespace

// ====================================================================================
// C ABI
// ====================================================================================
extern "C" merf_status merf_bundle_write(const char* dir, const merf_scene_desc* desc, const uint8_t* planes,
                                         const int32_t* block_index, const uint8_t* atlas, int64_t n_blocks,
                                         const uint32_t* occ_finest, const float* mlp) {
    if (!dir || !desc || !occ_finest || !mlp) return efail(MERF_EINVAL, "NULL argument");
    merf_status e = check_desc(desc);
    if (e) return e;
    const bool has_v = desc->L > 0, has_p = desc->R > 0;
    if ((has_p && !planes) || (has_v && (!block_index || n_blocks < 0 || (n_blocks > 0 && !atlas))))
        return efail(MERF_EINVAL, "NULL planes / block_index / atlas for the declared sources");
    if (has_v) {   // refuse a payload/manifest mismatch
        const int64_t slots = (int64_t)(desc->L / 8) * (desc->L / 8) * (desc->L / 8);
        for (int64_t i = 0; i < slots; i++)
            if (block_index[i] < -1 || block_index[i] >= n_blocks)
                return efail(MERF_EMISMATCH, "block_index[%lld] = %d outside [-1, n_blocks)", (long long)i, block_index[i]);
    }
    if (mkdir(dir, 0755) != 0 && errno != EEXIST) return efail(MERF_EIO, "%s: cannot create directory", dir);
    std::vector<Payload> pay;
    if (has_p)
        for (int a = 0; a < 3; a++)
            if (!encode_split(planes + (size_t)a * desc->R * desc->R * 8, desc->R, desc->R, "plane" + std::to_string(a), pay))
                return efail(MERF_EIO, "PNG encoding failed");
    if (has_v) {
        if (n_blocks > 0) {
            int w, h;
            atlas_raster_dims(n_blocks, w, h);
            std::vector<uint8_t> ras((size_t)w * h * 8, 0);
            atlas_to_raster(atlas, n_blocks, w, ras.data());
            if (!encode_split(ras.data(), w, h, "atlas", pay)) return efail(MERF_EIO, "PNG encoding failed");
        }
        const int64_t slots = (int64_t)(desc->L / 8) * (desc->L / 8) * (desc->L / 8);
        Payload b{"block_index.bin", std::vector<uint8_t>(slots * 4)};
        memcpy(b.bytes.data(), block_index, slots * 4);   // little-endian host
        pay.push_back(std::move(b));
    }
    const int Nf = desc->level_res[desc->n_levels - 1];
    const uint8_t* fine = reinterpret_cast<const uint8_t*>(occ_finest);
    for (int i = 0; i < desc->n_levels; i++) {
        const int N = desc->level_res[i];
        Payload o{"occupancy" + std::to_string(i) + ".bin", {}};
        if (N == Nf) {
            o.bytes.assign(fine, fine + occ_bytes(Nf));
            // bits past N^3 in the last byte are not cells: write them as 0
            const int64_t cells = (int64_t)N * N * N;
            if (cells % 8) o.bytes.back() &= uint8_t((1u << (cells % 8)) - 1u);
        } else {
            o.bytes = pool_bits(fine, Nf, N);
        }
        pay.push_back(std::move(o));
    }
    std::string man;
    char buf[256];
    man += "# MERF baked-scene bundle (PAPER.md Sec. 5.3); see include/merf.h merf_bundle_write\n";
    snprintf(buf, sizeof buf, "merf_bundle %d\nL %d\nR %d\nC %d\nblock_size 8\n", kVersion, desc->L, desc->R, desc->C);
    man += buf;
    man += "level_res";
    for (int i = 0; i < desc->n_levels; i++) man += " " + std::to_string(desc->level_res[i]);
    man += "\n";
    snprintf(buf, sizeof buf, "m_density %.9g\nm_appearance %.9g\nstep %.17g\nt_min %.9g\nalpha_skip %.9g\n",
             desc->m_density, desc->m_appearance, desc->step, desc->t_min, desc->alpha_skip);
    man += buf;
    snprintf(buf, sizeof buf, "source_mask %u\nn_blocks %lld\nbackground none\nmlp_dims 34 16 16 3\nmlp", desc->source_mask,
             (long long)n_blocks);
    man += buf;
    for (int i = 0; i < 883; i++) {
        snprintf(buf, sizeof buf, " %.9g", mlp[i]);
        man += buf;
    }
    man += "\n";
    for (auto& p : pay) {
        if (!write_file(join(dir, p.name), p.bytes.data(), p.bytes.size()))
            return efail(MERF_EIO, "%s: write failed", p.name.c_str());
        snprintf(buf, sizeof buf, "file %s %zu %08x\n", p.name.c_str(), p.bytes.size(),
                 (unsigned)crc32_z(0L, p.bytes.data(), p.bytes.size()));
        man += buf;
    }
    if (!write_file(join(dir, "manifest.txt"), man.data(), man.size())) return efail(MERF_EIO, "manifest write failed");
    return MERF_OK;
}

extern "C" merf_status merf_bundle_read(const char* dir, merf_scene_desc* desc, int64_t* n_blocks, uint8_t* planes,
                                        int32_t* block_index, uint8_t* atlas, uint32_t* occ_finest, float* mlp) {
    if (!dir || !desc || !n_blocks) return efail(MERF_EINVAL, "NULL argument");
    Manifest m;
    merf_status e = parse_manifest(dir, m);
    if (e) return e;
    *desc = m.desc;
    *n_blocks = m.n_blocks;
    if (!planes && !block_index && !atlas && !occ_finest && !mlp) return MERF_OK;   // query
    const bool has_v = m.desc.L > 0, has_p = m.desc.R > 0;
    if (!occ_finest || !mlp || (has_p && !planes) || (has_v && (!block_index || (m.n_blocks > 0 && !atlas))))
        return efail(MERF_EINVAL, "NULL output array for a stored payload");
    memcpy(mlp, m.mlp.data(), 883 * sizeof(float));
    if (has_p)
        for (int a = 0; a < 3; a++)
            if ((e = decode_split(dir, m, "plane" + std::to_string(a), m.desc.R, m.desc.R,
                                  planes + (size_t)a * m.desc.R * m.desc.R * 8)))
                return e;
    std::vector<uint8_t> f;
    if (has_v) {
        if (m.n_blocks > 0) {
            int w, h;
            atlas_raster_dims(m.n_blocks, w, h);
            std::vector<uint8_t> ras((size_t)w * h * 8);
            if ((e = decode_split(dir, m, "atlas", w, h, ras.data()))) return e;
            raster_to_atlas(ras.data(), m.n_blocks, w, atlas);
        }
        const int64_t slots = (int64_t)(m.desc.L / 8) * (m.desc.L / 8) * (m.desc.L / 8);
        if ((e = load_payload(dir, m, "block_index.bin", f))) return e;
        if ((int64_t)f.size() != slots * 4) return efail(MERF_EIO, "block_index.bin: size mismatch with L");
        memcpy(block_index, f.data(), f.size());
        for (int64_t i = 0; i < slots; i++)
            if (block_index[i] < -1 || block_index[i] >= m.n_blocks)
                return efail(MERF_EMISMATCH, "block_index.bin: entry %lld outside [-1, n_blocks)", (long long)i);
    }
    const int nl = m.desc.n_levels, Nf = m.desc.level_res[nl - 1];
    std::vector<uint8_t> fine;
    if ((e = load_payload(dir, m, "occupancy" + std::to_string(nl - 1) + ".bin", fine))) return e;
    if ((int64_t)fine.size() != occ_bytes(Nf)) return efail(MERF_EIO, "occupancy%d.bin: size mismatch with level_res", nl - 1);
    const size_t words = (size_t)(((int64_t)Nf * Nf * Nf + 31) / 32);
    memset(occ_finest, 0, words * 4);
    memcpy(occ_finest, fine.data(), fine.size());
    for (int i = 0; i < nl - 1; i++) {   // coarse levels must be the OR-pool of the finest
        if ((e = load_payload(dir, m, "occupancy" + std::to_string(i) + ".bin", f))) return e;
        if (f != pool_bits(fine.data(), Nf, m.desc.level_res[i]))
            return efail(MERF_EMISMATCH, "occupancy%d.bin is not the max-pool of the finest level", i);
    }
    return MERF_OK;
}

extern "C" merf_status merf_scene_load(const char* dir, int32_t device, merf_scene** out) {
    if (!dir || !out) return efail(MERF_EINVAL, "NULL argument");
    merf_scene_desc d;
    int64_t nb = 0;
    merf_status e = merf_bundle_read(dir, &d, &nb, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (e) return e;
    const int Nf = d.level_res[d.n_levels - 1];
    std::vector<uint8_t> planes(d.R ? (size_t)3 * d.R * d.R * 8 : 0);
    std::vector<int32_t> bidx(d.L ? (size_t)(d.L / 8) * (d.L / 8) * (d.L / 8) : 0);
    std::vector<uint8_t> atlas((size_t)nb * 729 * 8);
    std::vector<uint32_t> occ((size_t)(((int64_t)Nf * Nf * Nf + 31) / 32));
    std::vector<float> mlp(883);
    e = merf_bundle_read(dir, &d, &nb, planes.empty() ? nullptr : planes.data(), bidx.empty() ? nullptr : bidx.data(),
                         atlas.empty() ? nullptr : atlas.data(), occ.data(), mlp.data());
    if (e) return e;
    return merf_scene_upload(&d, planes.empty() ? nullptr : planes.data(), bidx.empty() ? nullptr : bidx.data(),
                             atlas.empty() ? nullptr : atlas.data(), nb, occ.data(), mlp.data(), device, out);
}

// Camera file: one camera per line (blank lines and '#' comments skipped), 20 numbers
//   W H fx fy cx cy  r00 r01 r02 t0  r10 r11 r12 t1  r20 r21 r22 t2  near far
// (camera-to-world rows [R | t], OpenCV axes, reading D18).  The rotation must be
// orthonormal with det +1 (|R R^T - I| <= 1e-6); far > near >= 0 (the renderer marches the
// contracted ray to the scene boundary; far is validated and otherwise unused).
extern "C" merf_status merf_cameras_read(const char* path, merf_camera* cams, int32_t max_cams, int32_t* n_cams,
                                         int32_t* widths, int32_t* heights) {
    if (!path || !n_cams) return efail(MERF_EINVAL, "NULL argument");
    std::vector<uint8_t> txt;
    if (!read_file(path, txt)) return efail(MERF_EIO, "%s: cannot read", path);
    txt.push_back(0);
    int n = 0, line_no = 0;
    std::string all((const char*)txt.data());
    size_t pos = 0;
    while (pos <= all.size()) {
        size_t nl = all.find('\n', pos);
        if (nl == std::string::npos) nl = all.size();
        std::string line = all.substr(pos, nl - pos);
        pos = nl + 1;
        line_no++;
        const size_t h = line.find('#');
        if (h != std::string::npos) line.resize(h);
        double v[21];
        int k = 0, off = 0;
        const char* q = line.c_str();
        while (k < 21 && sscanf(q, "%lf%n", &v[k], &off) == 1) {
            q += off;
            k++;
        }
        while (*q == ' ' || *q == '\t' || *q == '\r') q++;
        if (k == 0 && *q == 0) continue;
        if (k != 20 || *q != 0) return efail(MERF_EIO, "%s line %d: expected 20 numbers", path, line_no);
        if (v[0] < 1 || v[1] < 1 || v[0] != floor(v[0]) || v[1] != floor(v[1]))
            return efail(MERF_EIO, "%s line %d: width/height must be positive integers", path, line_no);
        if (!(v[2] > 0) || !(v[3] > 0)) return efail(MERF_EIO, "%s line %d: fx, fy must be > 0", path, line_no);
        if (!(v[18] >= 0) || !(v[19] > v[18])) return efail(MERF_EIO, "%s line %d: need far > near >= 0", path, line_no);
        double Rm[3][3];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) Rm[r][c] = v[6 + 4 * r + c];
        double err = 0.0;
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double s = 0.0;
                for (int c = 0; c < 3; c++) s += Rm[a][c] * Rm[b][c];
                err = fmax(err, fabs(s - (a == b ? 1.0 : 0.0)));
            }
        const double det = Rm[0][0] * (Rm[1][1] * Rm[2][2] - Rm[1][2] * Rm[2][1]) -
                           Rm[0][1] * (Rm[1][0] * Rm[2][2] - Rm[1][2] * Rm[2][0]) +
                           Rm[0][2] * (Rm[1][0] * Rm[2][1] - Rm[1][1] * Rm[2][0]);
        if (err > 1e-6 || det < 0) return efail(MERF_EIO, "%s line %d: rotation is not orthonormal (det +1)", path, line_no);
        if (cams) {
            if (n >= max_cams) return efail(MERF_EINVAL, "%s: more than max_cams = %d cameras", path, max_cams);
            for (int i = 0; i < 12; i++) cams[n].c2w[i] = v[6 + i];
            cams[n].fx = v[2];
            cams[n].fy = v[3];
            cams[n].cx = v[4];
            cams[n].cy = v[5];
            cams[n].t_near = v[18];
            if (widths) widths[n] = (int32_t)v[0];
            if (heights) heights[n] = (int32_t)v[1];
        }
        n++;
    }
    *n_cams = n;
    return MERF_OK;
}
