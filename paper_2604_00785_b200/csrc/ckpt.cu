// Record files of the sharded checkpoint (reference src/reliability.cpp:23-320) with the
// crc32 computed on the GPU over HBM. See ckpt.h for the format and the data flow.
//
// crc32 algebra (zlib's reflected CRC-32, polynomial 0xEDB88320). With the register form
// raw(r, M) (no pre/post inversion), zlib's crc32(c, M) = ~raw(~c, M), and
//   raw(r, A || B) = Z_|B|(raw(r, A)) ^ raw(0, B)
// where Z_L (feed L zero bytes) is linear over GF(2). So every 16-byte lane word, every
// 512-byte warp block and every 64 KB segment is hashed independently from r = 0 and the
// pieces are folded with Z: inside a warp by byte-sliced Z tables in shared memory, across
// segments on the host with byte-sliced Z tables (and 32x32 GF(2) matrices for odd lengths).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "../../include/b2moe.h"
#include "ckpt.h"

namespace b2 {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int64_t kSegBytes = 64 * 1024;          // one warp per segment
constexpr size_t kChunkBytes = 32u << 20;          // host <-> device streaming unit
static_assert(kChunkBytes % kSegBytes == 0, "chunks hold whole segments");
constexpr char kMagic[4] = {'O', 'P', 'T', 'T'};
constexpr uint32_t kVersion = 1;

// w[j][b]: raw(0, 16-byte word with byte b at position j, zeros elsewhere)
// z[l][k][b]: Z_{16 << l}(b << 8k), l = 0..5 (16..512 zero bytes)
struct CrcTables {
    uint32_t w[16][256];
    uint32_t z[6][4][256];
};
static_assert(sizeof(CrcTables) == 40960, "crc tables: 40 KB of shared memory");

__device__ CrcTables g_crc_tables;

struct HostCrc {
    uint32_t tab[256];
    uint32_t pow2[64][32];  // Z_{2^k} as 32 column images
    uint32_t seg[4][256];   // Z_{kSegBytes}, byte-sliced
    CrcTables dev;
    HostCrc() {
        for (uint32_t b = 0; b < 256; ++b) {
            uint32_t r = b;
            for (int i = 0; i < 8; ++i) r = (r & 1) ? (r >> 1) ^ kPoly : r >> 1;
            tab[b] = r;
        }
        for (int i = 0; i < 32; ++i) pow2[0][i] = zero_bytes(1u << i, 1);
        for (int k = 1; k < 64; ++k)
            for (int i = 0; i < 32; ++i) pow2[k][i] = apply(pow2[k - 1], apply(pow2[k - 1], 1u << i));
        for (int k = 0; k < 4; ++k)
            for (int b = 0; b < 256; ++b) seg[k][b] = shift((uint32_t)b << (8 * k), (uint64_t)kSegBytes);
        for (int j = 0; j < 16; ++j)
            for (int b = 0; b < 256; ++b) dev.w[j][b] = zero_bytes(tab[b], 15 - j);
        for (int l = 0; l < 6; ++l)
            for (int k = 0; k < 4; ++k)
                for (int b = 0; b < 256; ++b) dev.z[l][k][b] = zero_bytes((uint32_t)b << (8 * k), 16 << l);
    }
    uint32_t zero_bytes(uint32_t r, int n) const {
        for (int i = 0; i < n; ++i) r = tab[r & 0xff] ^ (r >> 8);
        return r;
    }
    static uint32_t apply(const uint32_t* m, uint32_t v) {  // branch-free GF(2) mat-vec
        uint32_t s = 0;
        for (int i = 0; i < 32; ++i) s ^= m[i] & (0u - ((v >> i) & 1u));
        return s;
    }
    uint32_t shift_seg(uint32_t r) const {
        return seg[0][r & 0xff] ^ seg[1][(r >> 8) & 0xff] ^ seg[2][(r >> 16) & 0xff] ^ seg[3][r >> 24];
    }
    uint32_t shift(uint32_t r, uint64_t n) const {
        for (int k = 0; n && r; ++k, n >>= 1)
            if (n & 1) r = apply(pow2[k], r);
        return r;
    }
};

const HostCrc& host_crc() {
    static const HostCrc h;
    return h;
}

// upload the tables once per device (the __device__ symbol has one instance per device)
void ensure_tables(int device) {
    static std::mutex mu;
    static uint64_t done = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (device < 64 && (done >> device) & 1) return;
    B2_CUDA(cudaMemcpyToSymbol(g_crc_tables, &host_crc().dev, sizeof(CrcTables)));
    if (device < 64) done |= 1ull << device;
}

__device__ __forceinline__ uint32_t zshift(const CrcTables& t, int l, uint32_t x) {
    return t.z[l][0][x & 0xff] ^ t.z[l][1][(x >> 8) & 0xff] ^ t.z[l][2][(x >> 16) & 0xff] ^ t.z[l][3][x >> 24];
}

__device__ __forceinline__ uint32_t word_crc(const CrcTables& t, uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) c ^= t.w[4 * q + k][(w[q] >> (8 * k)) & 0xff];
    return c;
}

template <bool ALIGNED>
__device__ __forceinline__ uint4 load16(const uint8_t* p) {
    if constexpr (ALIGNED) {
        uint4 v;
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
        return v;
    } else {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = (uint32_t)p[4 * q] | ((uint32_t)p[4 * q + 1] << 8) | ((uint32_t)p[4 * q + 2] << 16) |
                   ((uint32_t)p[4 * q + 3] << 24);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// out[s] = raw(0, bytes of segment s). One warp per 64 KB segment, persistent grid. Lane l
// owns the 16-byte words at 16 l + 512 k (coalesced 512-byte warp loads) and keeps its own
// register A_l = Z_512(A_l) ^ crc(word); at the segment end lane l's register still lacks
// the 16 (31 - l) bytes that follow its word in the last block, so
//   raw(0, segment) = XOR_l Z_{16 (31 - l)}(A_l)   (+ the sub-512-byte tail, lane 0).
// Per 512 bytes: 16 word-table + 4 shift-table lookups per lane, no shuffles.
template <bool ALIGNED>
__global__ void __launch_bounds__(256) crc32_segments_kernel(const uint8_t* __restrict__ p, int64_t n,
                                                            int64_t nseg, uint32_t* __restrict__ out) {
    __shared__ __align__(16) CrcTables t;
    {
        const uint4* src = reinterpret_cast<const uint4*>(&g_crc_tables);
        uint4* dst = reinterpret_cast<uint4*>(&t);
        for (int i = threadIdx.x; i < (int)(sizeof(CrcTables) / 16); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nseg; s += nwarps) {
        const int64_t base = s * kSegBytes;
        const int64_t len = min(kSegBytes, n - base);
        const int64_t blocks = len >> 9;
        const uint8_t* q = p + base + lane * 16;
        uint32_t a = 0;
        uint4 cur = blocks > 0 ? load16<ALIGNED>(q) : make_uint4(0, 0, 0, 0);
        for (int64_t b = 0; b < blocks; ++b) {
            const uint4 nxt = (b + 1 < blocks) ? load16<ALIGNED>(q + (b + 1) * 512) : cur;
            a = zshift(t, 5, a) ^ word_crc(t, cur);
            cur = nxt;
        }
        const int after = 31 - lane;  // Z_{16 * after} by its binary digits
#pragma unroll
        for (int l = 0; l < 5; ++l)
            if ((after >> l) & 1) a = zshift(t, l, a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a ^= __shfl_xor_sync(0xffffffffu, a, o);
        uint32_t acc = blocks > 0 ? a : 0;
        if (lane == 0) {
            for (int64_t i = blocks << 9; i < len; ++i) acc = t.w[15][(acc ^ p[base + i]) & 0xff] ^ (acc >> 8);
            out[s] = acc;
        }
    }
}

// RecordFileWriter::add_bf16 rounding (common.hpp:116-122): NaN stays quiet, else RNE
__global__ void f32_to_bf16_bits_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float f = in[i];
        const uint32_t u = __float_as_uint(f);
        out[i] = f != f ? (uint16_t)((u >> 16) | 0x0040u) : (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
    }
}

__global__ void bf16_bits_to_f32_kernel(const uint16_t* __restrict__ in, float* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __uint_as_float((uint32_t)in[i] << 16);
}

int elementwise_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

int current_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// segment crcs of n device bytes into dev_out (ceil(n / kSegBytes) entries)
void launch_crc_segments(const void* dev, int64_t n, uint32_t* dev_out, cudaStream_t st) {
    const int64_t nseg = (n + kSegBytes - 1) / kSegBytes;
    if (nseg == 0) return;
    const int grid = (int)std::min<int64_t>((nseg + 7) / 8, (int64_t)current_sms() * 5);
    const uint8_t* p = static_cast<const uint8_t*>(dev);
    if (((uintptr_t)p & 15) == 0)
        crc32_segments_kernel<true><<<grid, 256, 0, st>>>(p, n, nseg, dev_out);
    else
        crc32_segments_kernel<false><<<grid, 256, 0, st>>>(p, n, nseg, dev_out);
    B2_CUDA(cudaGetLastError());
}

// fold segment registers (each from r = 0) of an n-byte run into raw(0, run)
uint32_t fold_segments(const uint32_t* seg, int64_t n) {
    const HostCrc& h = host_crc();
    const int64_t nseg = (n + kSegBytes - 1) / kSegBytes;
    uint32_t r = 0;
    for (int64_t s = 0; s < nseg; ++s) {
        const int64_t len = std::min<int64_t>(kSegBytes, n - s * kSegBytes);
        r = (len == kSegBytes ? h.shift_seg(r) : h.shift(r, (uint64_t)len)) ^ seg[s];
    }
    return r;
}

void write_all(int fd, const void* p, size_t n, const std::string& path) {
    const char* c = static_cast<const char*>(p);
    while (n > 0) {
        const ssize_t w = ::write(fd, c, n);
        if (w < 0) throw IoError(path + ": write failed");
        c += w;
        n -= (size_t)w;
    }
}

void pread_all(int fd, void* p, size_t n, uint64_t off, const std::string& path) {
    char* c = static_cast<char*>(p);
    while (n > 0) {
        const ssize_t r = ::pread(fd, c, n, (off_t)off);
        if (r <= 0) throw IoError(path + ": read failed");
        c += r;
        n -= (size_t)r;
        off += (uint64_t)r;
    }
}

void put_u32(std::string& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back((char)((v >> (8 * i)) & 0xff));
}
void put_u64(std::string& b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back((char)((v >> (8 * i)) & 0xff));
}
uint32_t get_u32(const uint8_t* b) { return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24; }
uint64_t get_u64(const uint8_t* b) { return (uint64_t)get_u32(b) | (uint64_t)get_u32(b + 4) << 32; }

int64_t rec_numel(const std::vector<int64_t>& dims) {  // reliability.cpp:76-83
    int64_t n = 1;
    for (int64_t d : dims) {
        check(d >= 0, "record: negative dimension");
        n *= d;
    }
    return n;
}

}  // namespace

// pinned host double buffer + device staging double buffer + segment crc scratch
class Staging {
  public:
    explicit Staging(bool device_side) {
        for (int i = 0; i < 2; ++i) {
            B2_CUDA(cudaHostAlloc(&host[i], kChunkBytes, cudaHostAllocDefault));
            B2_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
            if (device_side) B2_CUDA(cudaMalloc(&dev[i], kChunkBytes));
        }
    }
    ~Staging() {
        for (int i = 0; i < 2; ++i) {
            if (host[i]) cudaFreeHost(host[i]);
            if (dev[i]) cudaFree(dev[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
        if (seg_dev) cudaFree(seg_dev);
        if (seg_host) cudaFreeHost(seg_host);
    }
    // room for n segment registers, device and pinned host
    void reserve_segs(int64_t n) {
        if (n <= seg_cap) return;
        if (seg_dev) cudaFree(seg_dev);
        if (seg_host) cudaFreeHost(seg_host);
        seg_cap = std::max<int64_t>(n, 1024);
        B2_CUDA(cudaMalloc((void**)&seg_dev, 4 * (size_t)seg_cap));
        B2_CUDA(cudaHostAlloc((void**)&seg_host, 4 * (size_t)seg_cap, cudaHostAllocDefault));
    }
    void* host[2] = {nullptr, nullptr};
    void* dev[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    uint32_t* seg_dev = nullptr;
    uint32_t* seg_host = nullptr;
    int64_t seg_cap = 0;
};

uint32_t crc_raw_update_host(uint32_t raw, const void* p, size_t n) {
    const HostCrc& h = host_crc();
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) raw = h.tab[(raw ^ b[i]) & 0xff] ^ (raw >> 8);
    return raw;
}

uint32_t crc_shift_host(uint32_t raw, uint64_t nbytes) { return host_crc().shift(raw, nbytes); }

uint32_t crc32_device(const void* dev, int64_t n, uint32_t crc_in, cudaStream_t st) {
    check(n >= 0 && (n == 0 || dev != nullptr), "crc32: bad buffer");
    int device = 0;
    B2_CUDA(cudaGetDevice(&device));
    ensure_tables(device);
    const int64_t nseg = (n + kSegBytes - 1) / kSegBytes;
    uint32_t* d = nullptr;
    std::vector<uint32_t> h((size_t)std::max<int64_t>(nseg, 1));
    if (nseg > 0) {
        B2_CUDA(cudaMallocAsync((void**)&d, 4 * (size_t)nseg, st));
        launch_crc_segments(dev, n, d, st);
        B2_CUDA(cudaMemcpyAsync(h.data(), d, 4 * (size_t)nseg, cudaMemcpyDeviceToHost, st));
        B2_CUDA(cudaFreeAsync(d, st));
        B2_CUDA(cudaStreamSynchronize(st));
    }
    const uint32_t r = host_crc().shift(~crc_in, (uint64_t)n) ^ fold_segments(h.data(), n);
    return ~r;
}

void launch_f32_to_bf16_bits(const float* in, uint16_t* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    f32_to_bf16_bits_kernel<<<elementwise_grid(n), 256, 0, st>>>(in, out, n);
    B2_CUDA(cudaGetLastError());
}

void launch_bf16_bits_to_f32(const uint16_t* in, float* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    bf16_bits_to_f32_kernel<<<elementwise_grid(n), 256, 0, st>>>(in, out, n);
    B2_CUDA(cudaGetLastError());
}

// ---- writer -----------------------------------------------------------------------------

RecordWriter::RecordWriter(int device, cudaStream_t st, const std::string& path)
    : device_(device), st_(st), path_(path) {
    B2_CUDA(cudaSetDevice(device_));
    ensure_tables(device_);
    fd_ = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd_ < 0) throw IoError(path + ": cannot create");
    stage_ = new Staging(false);
    const char zeros[12] = {0};  // header: patched by finish()
    write_all(fd_, zeros, sizeof zeros, path_);
}

RecordWriter::~RecordWriter() {
    if (fd_ >= 0) ::close(fd_);
    delete stage_;
}

void RecordWriter::put_host(const void* p, size_t n) {
    write_all(fd_, p, n, path_);
    body_raw_ = crc_raw_update_host(body_raw_, p, n);
    body_len_ += n;
}

void RecordWriter::put_device(const void* dev, size_t n) {
    if (n == 0) return;
    const int64_t nseg = ((int64_t)n + kSegBytes - 1) / kSegBytes;
    stage_->reserve_segs(nseg);
    launch_crc_segments(dev, (int64_t)n, stage_->seg_dev, st_);
    B2_CUDA(cudaMemcpyAsync(stage_->seg_host, stage_->seg_dev, 4 * (size_t)nseg, cudaMemcpyDeviceToHost, st_));
    // payload: device -> pinned (async) overlapped with pinned -> file of the previous chunk
    const char* src = static_cast<const char*>(dev);
    const size_t nchunks = (n + kChunkBytes - 1) / kChunkBytes;
    size_t prev_len = 0;
    for (size_t i = 0; i <= nchunks; ++i) {
        const int b = (int)(i & 1);
        if (i < nchunks) {
            const size_t len = std::min(kChunkBytes, n - i * kChunkBytes);
            B2_CUDA(cudaMemcpyAsync(stage_->host[b], src + i * kChunkBytes, len, cudaMemcpyDeviceToHost, st_));
            B2_CUDA(cudaEventRecord(stage_->ev[b], st_));
            if (i > 0) {
                B2_CUDA(cudaEventSynchronize(stage_->ev[b ^ 1]));
                write_all(fd_, stage_->host[b ^ 1], prev_len, path_);
            }
            prev_len = len;
        } else {
            B2_CUDA(cudaEventSynchronize(stage_->ev[b ^ 1]));
            write_all(fd_, stage_->host[b ^ 1], prev_len, path_);
        }
    }
    B2_CUDA(cudaStreamSynchronize(st_));
    const uint32_t payload = fold_segments(stage_->seg_host, (int64_t)n);
    body_raw_ = crc_shift_host(body_raw_, n) ^ payload;
    body_len_ += n;
}

void RecordWriter::add(const std::string& name, RecDtype dt, const std::vector<int64_t>& dims, const void* src,
                       int src_dtype) {
    check(!done_, "record writer: already finished");
    check(src_dtype == B2_F32 || src_dtype == B2_BF16, "record writer: source dtype must be f32 or bf16");
    check(dims.size() <= 8, "record '" + name + "': too many dimensions");
    const int64_t n = rec_numel(dims);
    check(n == 0 || src != nullptr, "record '" + name + "': null source");
    B2_CUDA(cudaSetDevice(device_));
    std::string h;
    put_u32(h, (uint32_t)name.size());
    h.append(name);
    put_u32(h, (uint32_t)dt);
    put_u32(h, (uint32_t)dims.size());
    for (int64_t d : dims) put_u64(h, (uint64_t)d);
    put_host(h.data(), h.size());
    const int src_rec = src_dtype == B2_F32 ? 0 : 1;
    if ((int)dt == src_rec) {
        put_device(src, (size_t)n * (dt == RecDtype::f32 ? 4 : 2));
    } else {  // convert in HBM first
        void* tmp = nullptr;
        const size_t bytes = (size_t)n * (dt == RecDtype::f32 ? 4 : 2);
        B2_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(bytes, 16), st_));
        if (dt == RecDtype::bf16)
            launch_f32_to_bf16_bits(static_cast<const float*>(src), static_cast<uint16_t*>(tmp), n, st_);
        else
            launch_bf16_bits_to_f32(static_cast<const uint16_t*>(src), static_cast<float*>(tmp), n, st_);
        put_device(tmp, bytes);
        B2_CUDA(cudaFreeAsync(tmp, st_));
    }
    ++count_;
}

RecordWriter::Written RecordWriter::finish() {
    check(!done_, "record writer: already finished");
    std::string head;
    head.append(kMagic, 4);
    put_u32(head, kVersion);
    put_u32(head, count_);
    const uint32_t raw = crc_shift_host(crc_raw_update_host(0xffffffffu, head.data(), head.size()), body_len_) ^ body_raw_;
    const uint32_t crc = ~raw;
    std::string foot;
    put_u32(foot, crc);
    write_all(fd_, foot.data(), foot.size(), path_);
    if (::pwrite(fd_, head.data(), head.size(), 0) != (ssize_t)head.size()) throw IoError(path_ + ": write failed");
    if (::fsync(fd_) != 0) throw IoError(path_ + ": fsync failed");
    ::close(fd_);
    fd_ = -1;
    done_ = true;
    return Written{(int64_t)(head.size() + body_len_ + foot.size()), crc};
}

// ---- reader -----------------------------------------------------------------------------

RecordFile::RecordFile(int device, cudaStream_t st, const std::string& path)
    : device_(device), st_(st), path_(path) {
    B2_CUDA(cudaSetDevice(device_));
    ensure_tables(device_);
    auto bad = [&](const std::string& why) { return IoError(path + ": " + why); };
    fd_ = ::open(path.c_str(), O_RDONLY);
    if (fd_ < 0) throw IoError(path + ": cannot open");
    struct stat sb;
    if (::fstat(fd_, &sb) != 0) throw bad("cannot stat");
    size_ = (uint64_t)sb.st_size;
    if (size_ < 16) throw bad("truncated header");
    uint8_t head[12];
    pread_all(fd_, head, 12, 0, path_);
    if (std::memcmp(head, kMagic, 4) != 0) throw bad("bad magic");
    if (get_u32(head + 4) != kVersion) throw bad("unsupported version");

    // checksum over everything before the footer: file -> pinned -> HBM -> GPU crc
    stage_ = new Staging(true);
    const uint64_t body = size_ - 4;
    const int64_t nseg = (int64_t)((body + kSegBytes - 1) / kSegBytes);
    stage_->reserve_segs(nseg);
    const size_t nchunks = (size_t)((body + kChunkBytes - 1) / kChunkBytes);
    for (size_t i = 0; i < nchunks; ++i) {
        const int b = (int)(i & 1);
        const size_t len = (size_t)std::min<uint64_t>(kChunkBytes, body - i * kChunkBytes);
        if (i >= 2) B2_CUDA(cudaEventSynchronize(stage_->ev[b]));  // pinned + device buffer b free again
        pread_all(fd_, stage_->host[b], len, (uint64_t)i * kChunkBytes, path_);
        B2_CUDA(cudaMemcpyAsync(stage_->dev[b], stage_->host[b], len, cudaMemcpyHostToDevice, st_));
        launch_crc_segments(stage_->dev[b], (int64_t)len, stage_->seg_dev + i * (kChunkBytes / kSegBytes), st_);
        B2_CUDA(cudaEventRecord(stage_->ev[b], st_));
    }
    B2_CUDA(cudaMemcpyAsync(stage_->seg_host, stage_->seg_dev, 4 * (size_t)std::max<int64_t>(nseg, 0),
                            cudaMemcpyDeviceToHost, st_));
    B2_CUDA(cudaStreamSynchronize(st_));
    const uint32_t crc = ~(crc_shift_host(0xffffffffu, body) ^ fold_segments(stage_->seg_host, (int64_t)body));
    uint8_t foot[4];
    pread_all(fd_, foot, 4, body, path_);
    if (crc != get_u32(foot)) throw bad("checksum mismatch");

    // record headers (reliability.cpp:281-318): same bounds, same order
    const uint32_t count = get_u32(head + 8);
    uint64_t off = 12;
    auto need = [&](uint64_t n) {
        if (body - off < n) throw bad("truncated record");
    };
    std::vector<uint8_t> buf;
    auto take = [&](uint64_t n) {
        need(n);
        buf.resize((size_t)std::max<uint64_t>(n, 1));
        if (n) pread_all(fd_, buf.data(), (size_t)n, off, path_);
        off += n;
        return buf.data();
    };
    recs_.reserve(count);
    for (uint32_t r = 0; r < count; ++r) {
        RecordInfo rec;
        const uint32_t name_len = get_u32(take(4));
        if (name_len > 4096) throw bad("oversized record name");
        const uint8_t* nm = take(name_len);
        rec.name.assign(reinterpret_cast<const char*>(nm), name_len);
        const uint8_t* dn = take(8);
        const uint32_t dt = get_u32(dn), nd = get_u32(dn + 4);
        if (dt > 1) throw bad("unknown dtype");
        rec.dtype = (RecDtype)dt;
        if (nd > 8) throw bad("too many dimensions");
        const uint8_t* dd = take((uint64_t)nd * 8);
        for (uint32_t d = 0; d < nd; ++d) rec.dims.push_back((int64_t)get_u64(dd + 8 * d));
        rec.numel = rec_numel(rec.dims);
        const uint64_t payload = (uint64_t)rec.numel * (rec.dtype == RecDtype::f32 ? 4 : 2);
        need(payload);
        rec.offset = off;
        off += payload;
        recs_.push_back(std::move(rec));
    }
    if (off != body) throw bad("trailing bytes after last record");
}

RecordFile::~RecordFile() {
    if (fd_ >= 0) ::close(fd_);
    delete stage_;
}

int RecordFile::find(const std::string& name) const {
    for (size_t i = 0; i < recs_.size(); ++i)
        if (recs_[i].name == name) return (int)i;
    return -1;
}

void RecordFile::read(int i, int64_t b, int64_t e, void* dst, int dst_dtype) {
    check(i >= 0 && i < (int)recs_.size(), "record file: record index out of range");
    const RecordInfo& r = recs_[(size_t)i];
    check(0 <= b && b <= e && e <= r.numel, "record '" + r.name + "': element range out of bounds");
    check(dst_dtype == B2_F32 || dst_dtype == B2_BF16, "record file: destination dtype must be f32 or bf16");
    if (e == b) return;
    B2_CUDA(cudaSetDevice(device_));
    const size_t es = r.dtype == RecDtype::f32 ? 4 : 2;
    const size_t n = (size_t)(e - b) * es;
    const bool same = (dst_dtype == B2_F32) == (r.dtype == RecDtype::f32);
    char* out = static_cast<char*>(dst);
    void* tmp = nullptr;
    if (!same) {
        B2_CUDA(cudaMallocAsync(&tmp, n, st_));
        out = static_cast<char*>(tmp);
    }
    const size_t nchunks = (n + kChunkBytes - 1) / kChunkBytes;
    for (size_t c = 0; c < nchunks; ++c) {
        const int k = (int)(c & 1);
        const size_t len = std::min(kChunkBytes, n - c * kChunkBytes);
        if (c >= 2) B2_CUDA(cudaEventSynchronize(stage_->ev[k]));
        pread_all(fd_, stage_->host[k], len, r.offset + (uint64_t)b * es + c * kChunkBytes, path_);
        B2_CUDA(cudaMemcpyAsync(out + c * kChunkBytes, stage_->host[k], len, cudaMemcpyHostToDevice, st_));
        B2_CUDA(cudaEventRecord(stage_->ev[k], st_));
    }
    if (!same) {
        if (r.dtype == RecDtype::bf16)
            launch_bf16_bits_to_f32(static_cast<const uint16_t*>(tmp), static_cast<float*>(dst), e - b, st_);
        else
            launch_f32_to_bf16_bits(static_cast<const float*>(tmp), static_cast<uint16_t*>(dst), e - b, st_);
        B2_CUDA(cudaFreeAsync(tmp, st_));
    }
    B2_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace b2
