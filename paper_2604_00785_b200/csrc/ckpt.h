// Sharded checkpoint record files on B200.
//
// Format: the reference's record file (include/optimus/reliability.hpp:33-70,
// src/reliability.cpp:23-31): "OPTT", u32 version 1, u32 record count, per record
// {u32 name length, name, u32 dtype (0 f32, 1 bf16), u32 ndim, u64 dims, little-endian
// payload}, then the zlib crc32 of everything before the footer.
//
// B200 shape: payloads never leave HBM until they are written. The crc32 of every
// payload is computed on the GPU over HBM (64 KB segments, one warp each, combined on
// the host with GF(2) shift operators), the payload bytes stream device -> pinned host ->
// file in double-buffered 32 MB chunks, and only the record headers are built on the
// host. Reading validates the whole file the same way (file -> pinned -> HBM staging ->
// GPU crc) before a single record is handed out, then copies any element range of a
// record straight into device memory.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "b2_common.cuh"

namespace b2 {

struct IoError : Error {
    explicit IoError(const std::string& m) : Error(5, m) {}
};

enum class RecDtype : uint32_t { f32 = 0, bf16 = 1 };

// zlib-compatible crc32 continuation over device bytes (crc_in = 0 starts a new one)
uint32_t crc32_device(const void* dev, int64_t n, uint32_t crc_in, cudaStream_t st);
// host helpers of the same crc (register form, no pre/post inversion)
uint32_t crc_raw_update_host(uint32_t raw, const void* p, size_t n);
uint32_t crc_shift_host(uint32_t raw, uint64_t nbytes);  // feed nbytes zero bytes

// dtype conversions with the reference's rounding (common.hpp:116-126)
void launch_f32_to_bf16_bits(const float* in, uint16_t* out, int64_t n, cudaStream_t st);
void launch_bf16_bits_to_f32(const uint16_t* in, float* out, int64_t n, cudaStream_t st);

class Staging;  // pinned double buffer

// RecordFileWriter (reliability.hpp:47-71): records stream to the file as they are added;
// finish() patches the count into the header, appends the crc footer and fsyncs.
class RecordWriter {
  public:
    RecordWriter(int device, cudaStream_t st, const std::string& path);
    ~RecordWriter();
    // src: device pointer of prod(dims) elements of src_dtype (B2_F32 / B2_BF16)
    void add(const std::string& name, RecDtype dt, const std::vector<int64_t>& dims, const void* src,
             int src_dtype);
    struct Written {
        int64_t bytes = 0;
        uint32_t crc = 0;
    };
    Written finish();

  private:
    void put_host(const void* p, size_t n);
    void put_device(const void* dev, size_t n);
    int device_;
    cudaStream_t st_;
    std::string path_;
    int fd_ = -1;
    uint32_t count_ = 0;
    uint32_t body_raw_ = 0;  // crc register of the body from 0
    uint64_t body_len_ = 0;
    Staging* stage_ = nullptr;
    bool done_ = false;
};

struct RecordInfo {
    std::string name;
    RecDtype dtype = RecDtype::f32;
    std::vector<int64_t> dims;
    int64_t numel = 0;
    uint64_t offset = 0;  // payload offset in the file
};

// read_record_file (reliability.cpp:272-320): the constructor validates magic, version,
// crc and every record bound (same checks, same messages) before anything is read out.
class RecordFile {
  public:
    RecordFile(int device, cudaStream_t st, const std::string& path);
    ~RecordFile();
    const std::vector<RecordInfo>& records() const { return recs_; }
    int find(const std::string& name) const;  // -1 if absent
    // elements [b, e) of record i into device memory dst (dst_dtype B2_F32 / B2_BF16)
    void read(int i, int64_t b, int64_t e, void* dst, int dst_dtype);

  private:
    int device_;
    cudaStream_t st_;
    std::string path_;
    int fd_ = -1;
    uint64_t size_ = 0;
    std::vector<RecordInfo> recs_;
    Staging* stage_ = nullptr;
};

}  // namespace b2
