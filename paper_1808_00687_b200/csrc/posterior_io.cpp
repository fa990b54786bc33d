// posterior_io.cpp -- POST1 posterior files (reference posteriors.py:147-217) read straight into
// a caller buffer: the decoder's page-locked table, so a file's rows reach the GPU (read
// zero-copy by the kernel) without a pageable staging copy.
//
// POST1 = "POST1" + uint32 frames, columns, blank column (little-endian) + frames x columns
// little-endian float64, nothing after.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/wfst_b200.h"

int wb_internal_set_error(int code, const char *msg);

namespace {

static_assert(sizeof(double) == 8, "POST1 stores IEEE binary64");

struct File {
    FILE *f = nullptr;
    explicit File(const char *path) : f(std::fopen(path, "rb")) {}
    ~File() { if (f) std::fclose(f); }
};

int header(File &fh, const char *path, uint32_t h[3]) {
    if (!fh.f) return wb_internal_set_error(WB_ERR_VALUE, (std::string("cannot open ") + path).c_str());
    char magic[5];
    if (std::fread(magic, 1, 5, fh.f) != 5 || std::memcmp(magic, "POST1", 5) != 0)
        return wb_internal_set_error(WB_ERR_VALUE, "not a POST1 file");
    unsigned char b[12];
    if (std::fread(b, 1, 12, fh.f) != 12)
        return wb_internal_set_error(WB_ERR_VALUE, "binary posterior data truncated before header");
    for (int k = 0; k < 3; ++k)
        h[k] = (uint32_t)b[4 * k] | (uint32_t)b[4 * k + 1] << 8 | (uint32_t)b[4 * k + 2] << 16 |
               (uint32_t)b[4 * k + 3] << 24;
    std::fseek(fh.f, 0, SEEK_END);
    const long long size = std::ftell(fh.f), want = 17 + 8ll * h[0] * h[1];
    if (size != want)
        return wb_internal_set_error(WB_ERR_VALUE, ("binary posterior data has " + std::to_string(size) +
                                                    " bytes, expected " + std::to_string(want)).c_str());
    if (h[1] < 1 || h[2] >= h[1])
        return wb_internal_set_error(WB_ERR_VALUE, "blank column out of range");
    std::fseek(fh.f, 17, SEEK_SET);
    return WB_OK;
}

}  // namespace

extern "C" {

int wb_post1_info(const char *path, int32_t *num_frames, int32_t *num_cols, int32_t *blank_col) {
    if (!path || !num_frames || !num_cols || !blank_col) return wb_internal_set_error(WB_ERR_VALUE, "null argument");
    File fh(path);
    uint32_t h[3];
    if (int rc = header(fh, path, h)) return rc;
    *num_frames = (int32_t)h[0];
    *num_cols = (int32_t)h[1];
    *blank_col = (int32_t)h[2];
    return WB_OK;
}

int wb_post1_read(const char *path, double *dst, int64_t dst_ld) {
    if (!path || !dst) return wb_internal_set_error(WB_ERR_VALUE, "null argument");
    File fh(path);
    uint32_t h[3];
    if (int rc = header(fh, path, h)) return rc;
    if (dst_ld < (int64_t)h[1]) return wb_internal_set_error(WB_ERR_VALUE, "row stride below the column count");
    const size_t cols = h[1];
    if (dst_ld == (int64_t)cols) {   // one read of the whole matrix into the (pinned) table
        if (std::fread(dst, 8, cols * h[0], fh.f) != cols * h[0])
            return wb_internal_set_error(WB_ERR_VALUE, "short read");
    } else {
        for (uint32_t r = 0; r < h[0]; ++r)
            if (std::fread(dst + (size_t)r * dst_ld, 8, cols, fh.f) != cols)
                return wb_internal_set_error(WB_ERR_VALUE, "short read");
    }
    return WB_OK;
}

}  // extern "C"
