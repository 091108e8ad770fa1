// corpus.cu -- corpus emission on the device.
//
// write_corpus (engine.cpp:236-259) prints one walk per line, ids separated
// by single spaces, '\n' terminated, plus <path>.stats.jsonl. Here the
// integer-to-text formatting runs on the GPU over the walk buffer still in
// HBM: a length pass (digits + separators per row), a 64-bit exclusive scan
// for byte offsets, a write pass, then the text streams to the file through
// a pinned double buffer (D2H of chunk i+1 overlaps fwrite of chunk i).
#include <cub/cub.cuh>

#include <cstdio>
#include <string>

#include "internal.h"
#include "jsonfmt.h"
#include "exact.h"
#include "walk.h"

namespace mhw {

namespace {

__device__ __forceinline__ uint32_t ndigits(uint32_t x) {
    uint32_t d = 1;
    while (x >= 10) {
        x /= 10;
        ++d;
    }
    return d;
}

__global__ void k_text_len(const uint32_t* __restrict__ rows, uint32_t stride, const uint32_t* __restrict__ lens,
                           uint64_t n_rows, uint64_t* __restrict__ out) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n_rows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        if (r == n_rows) {
            out[r] = 0;
            continue;
        }
        const uint32_t* w = rows + r * stride;
        const uint32_t len = lens[r];
        uint64_t bytes = len;  // len - 1 spaces + 1 newline
        for (uint32_t i = 0; i < len; ++i) bytes += ndigits(w[i]);
        out[r] = bytes;
    }
}

__global__ void k_text_write(const uint32_t* __restrict__ rows, uint32_t stride, const uint32_t* __restrict__ lens,
                             const uint64_t* __restrict__ off, uint64_t n_rows, char* __restrict__ text) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t* w = rows + r * stride;
        const uint32_t len = lens[r];
        char* p = text + off[r];
        for (uint32_t i = 0; i < len; ++i) {
            if (i) *p++ = ' ';
            uint32_t x = w[i];
            const uint32_t nd = ndigits(x);
            for (uint32_t k = nd; k-- > 0;) {
                p[k] = (char)('0' + x % 10);
                x /= 10;
            }
            p += nd;
        }
        *p = '\n';
    }
}

unsigned grid_for(uint64_t work) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t g = (work + 255) / 256;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, (uint64_t)sms * 16));
}

}  // namespace

void session_write_corpus(Session& s, const char* path, const mhw_walk_stats& st) {
    DeviceGuard dg(s.g->device);
    cudaStream_t cs = s.stream;
    const uint64_t rows = s.rows;
    DBuf<uint64_t> len(rows + 1), off(rows + 1);
    k_text_len<<<grid_for(rows + 1), 256, 0, cs>>>(s.out.p, s.stride, s.lens.p, rows, len.p);
    size_t bytes = 0;
    MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.p, off.p, (int64_t)rows + 1, cs));
    DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
    MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, len.p, off.p, (int64_t)rows + 1, cs));
    uint64_t total = 0;
    MHW_CK(cudaMemcpyAsync(&total, off.p + rows, 8, cudaMemcpyDeviceToHost, cs));
    MHW_CK(cudaStreamSynchronize(cs));
    DBuf<char> text(std::max<uint64_t>(total, 1));
    if (rows) k_text_write<<<grid_for(rows), 256, 0, cs>>>(s.out.p, s.stride, s.lens.p, off.p, rows, text.p);
    MHW_CK(cudaGetLastError());
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(MHW_ERR_IO, std::string("cannot open for writing: ") + path);
    const uint64_t chunk = 64ull << 20;
    char* stage[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool ok = true;
    try {
        for (int i = 0; i < 2; ++i) {
            MHW_CK(cudaMallocHost(&stage[i], chunk));
            MHW_CK(cudaEventCreate(&ev[i]));
        }
        const uint64_t n_chunks = (total + chunk - 1) / chunk;
        auto issue = [&](uint64_t c) {
            const uint64_t b = c * chunk, n = std::min(chunk, total - b);
            MHW_CK(cudaMemcpyAsync(stage[c & 1], text.p + b, n, cudaMemcpyDeviceToHost, cs));
            MHW_CK(cudaEventRecord(ev[c & 1], cs));
        };
        if (n_chunks) issue(0);
        for (uint64_t c = 0; c < n_chunks && ok; ++c) {
            MHW_CK(cudaEventSynchronize(ev[c & 1]));
            if (c + 1 < n_chunks) issue(c + 1);  // next D2H overlaps this fwrite
            const uint64_t n = std::min(chunk, total - c * chunk);
            ok = std::fwrite(stage[c & 1], 1, n, f) == n;
        }
        MHW_CK(cudaStreamSynchronize(cs));
    } catch (...) {
        std::fclose(f);
        for (int i = 0; i < 2; ++i) {
            if (stage[i]) cudaFreeHost(stage[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
        throw;
    }
    for (int i = 0; i < 2; ++i) {
        cudaFreeHost(stage[i]);
        cudaEventDestroy(ev[i]);
    }
    if (std::fclose(f) != 0 || !ok) throw Error(MHW_ERR_IO, std::string("write failed: ") + path);
    const std::string side = std::string(path) + ".stats.jsonl";
    FILE* sf = std::fopen(side.c_str(), "wb");
    if (!sf) throw Error(MHW_ERR_IO, "cannot open for writing: " + side);
    const std::string line = stats_line(st);
    const bool sok = std::fwrite(line.data(), 1, line.size(), sf) == line.size();
    if (std::fclose(sf) != 0 || !sok) throw Error(MHW_ERR_IO, "write failed: " + side);
}

}  // namespace mhw
