// checkpoint.cu — checkpoint ingest / egress for a resident session
// (save_checkpoint / load_checkpoint, checkpoint.hpp:38-92).
//
// File format (the reference's, byte for byte): "GPILE", version u32 = 1,
// count u64, bbox 6 x f64 (min xyz, max xyz), then count records of 11
// little-endian f32 (mu xyz, log-scale xyz, quat wxyz, raw alpha). The record
// is the C-ABI's record layout, so the payload moves between the file and
// HBM through one pinned host buffer and the device transpose (layout.cu):
// no per-primitive host work.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/gpile_b200.h"
#include "common.cuh"

namespace {

constexpr char kMagic[5] = {'G', 'P', 'I', 'L', 'E'};
constexpr uint32_t kVersion = 1;

struct Pinned {
    void* p = nullptr;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

}  // namespace

extern "C" {

uint64_t gpk_checkpoint_bytes(uint64_t count) { return 5 + 4 + 8 + 6 * 8 + count * 11 * 4; }

int gpk_save_checkpoint(gpk_session* s, const char* path) {
    if (!s || !path) return gpk::set_last_error(GPK_ERR_INVALID_ARGUMENT, "save_checkpoint: null argument");
    uint64_t n = 0;
    gpk_bounds bb;
    int st = gpk_gaussian_count(s, &n);
    if (st == GPK_OK) st = gpk_get_bounds(s, &bb);
    if (st != GPK_OK) return st;
    Pinned buf;
    if (n && cudaMallocHost(&buf.p, n * 44) != cudaSuccess)
        return gpk::set_last_error(GPK_ERR_OUT_OF_MEMORY, "save_checkpoint: pinned buffer");
    if (n && (st = gpk_get_gaussians(s, static_cast<float*>(buf.p))) != GPK_OK) return st;
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) return gpk::set_last_error(GPK_ERR_LOAD, std::string("save_checkpoint: cannot open ") + path);
    const double box[6] = {bb.min[0], bb.min[1], bb.min[2], bb.max[0], bb.max[1], bb.max[2]};
    bool ok = std::fwrite(kMagic, 1, 5, out.f) == 5 && std::fwrite(&kVersion, 4, 1, out.f) == 1 &&
              std::fwrite(&n, 8, 1, out.f) == 1 && std::fwrite(box, 8, 6, out.f) == 6 &&
              (n == 0 || std::fwrite(buf.p, 44, n, out.f) == n);
    ok = (std::fclose(out.f) == 0) && ok;
    out.f = nullptr;
    if (!ok) return gpk::set_last_error(GPK_ERR_LOAD, std::string("save_checkpoint: write failed for ") + path);
    return GPK_OK;
}

int gpk_load_checkpoint(gpk_session* s, const char* path) {
    if (!s || !path) return gpk::set_last_error(GPK_ERR_INVALID_ARGUMENT, "load_checkpoint: null argument");
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) return gpk::set_last_error(GPK_ERR_LOAD, std::string("load_checkpoint: cannot open ") + path);
    char magic[5];
    if (std::fread(magic, 1, 5, in.f) != 5 || std::memcmp(magic, kMagic, 5) != 0)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER, std::string("load_checkpoint: bad magic in ") + path);
    uint32_t version = 0;
    if (std::fread(&version, 4, 1, in.f) != 1)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER, "unexpected end of file");
    if (version != kVersion)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER,
                                   "load_checkpoint: unsupported version " + std::to_string(version));
    uint64_t n = 0;
    if (std::fread(&n, 8, 1, in.f) != 1)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER, "unexpected end of file");
    double box[6];
    if (std::fread(box, 8, 6, in.f) != 6)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER, "load_checkpoint: truncated header");
    // the payload must be all there before anything is allocated for it
    const long here = std::ftell(in.f);
    std::fseek(in.f, 0, SEEK_END);
    const long end = std::ftell(in.f);
    std::fseek(in.f, here, SEEK_SET);
    const uint64_t avail = end > here ? (uint64_t)(end - here) / 44 : 0;
    if (avail < n)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER,
                                   "load_checkpoint: truncated record " + std::to_string(avail));
    Pinned buf;
    if (n && cudaMallocHost(&buf.p, n * 44) != cudaSuccess)
        return gpk::set_last_error(GPK_ERR_OUT_OF_MEMORY, "load_checkpoint: pinned buffer");
    if (n && std::fread(buf.p, 44, n, in.f) != n)
        return gpk::set_last_error(GPK_ERR_CORRUPT_CONTAINER,
                                   "load_checkpoint: truncated record " + std::to_string(avail));
    const gpk_bounds bb{{box[0], box[1], box[2]}, {box[3], box[4], box[5]}};
    return gpk_set_gaussians(s, n, static_cast<const float*>(buf.p), &bb);
}

}  // extern "C"
