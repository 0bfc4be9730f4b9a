// format.h -- the runtime's own CDM1 container parser (host side).
//
// Layout (the paper leaves it unspecified, SPEC.md:99 / SURVEY App. A):
//   header 64 B: magic "CDM1", u16 version=1, u16 n_nodes, u16 n_streams, u8 dtype, u8 pad, u32 width,
//                u64 rows, u64 payload_bytes, u64 offsets_bytes, u64 total_bytes, u64 cascade_hash,
//                u64 chunk_id
//   nodes, 32 B each, depth-first preorder: u8 codec, u8 n_children, u16 stream (Raw), u32 elem_bytes
//                (Raw), u64 n (elements decoded by this node), 16 B codec params
//   stream table, 16 B each: u64 offset (from chunk start, 16-aligned), u64 bytes
//   streams, zero padded to a 16-byte multiple plus 16 slack bytes.
#pragma once
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace cdm {

enum Codec : uint8_t { RAW = 0, BITPACK = 1, DICT = 2, FLOAT2INT = 3, DELTA = 4, RLE = 5, LZ4 = 6, STR = 7, ANS = 8, DSTRIDE = 9, STRDICT = 10 };
enum DType : uint8_t { T_I32 = 0, T_I64 = 1, T_F64 = 2, T_FIXED = 3, T_VARBYTES = 4 };

constexpr uint32_t kMagic = 0x314D4443u;  // "CDM1"
constexpr uint32_t kHeaderBytes = 64;
constexpr uint32_t kNodeBytes = 32;
constexpr uint32_t kStreamBytes = 16;

struct Node {
  uint8_t codec = 0, nchild = 0;
  uint16_t stream = 0xFFFF;
  uint32_t elem_bytes = 0;
  uint64_t n = 0;
  uint8_t params[16] = {};
  // decoded views of params
  uint32_t w() const { return params[0]; }
  uint64_t u64_at8() const { uint64_t v; std::memcpy(&v, params + 8, 8); return v; }
  uint32_t u32_at0() const { uint32_t v; std::memcpy(&v, params, 4); return v; }
  uint32_t u32_at4() const { uint32_t v; std::memcpy(&v, params + 4, 4); return v; }
};

struct Stream {
  uint64_t offset = 0, bytes = 0;
};

struct Chunk {
  uint8_t dtype = 0;
  uint32_t width = 0;
  uint64_t rows = 0, payload_bytes = 0, offsets_bytes = 0, total_bytes = 0, cascade_hash = 0, chunk_id = 0;
  std::vector<Node> nodes;
  std::vector<Stream> streams;
};

inline uint64_t rd64(const uint8_t* p) { uint64_t v; std::memcpy(&v, p, 8); return v; }
inline uint32_t rd32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }
inline uint16_t rd16(const uint8_t* p) { uint16_t v; std::memcpy(&v, p, 2); return v; }

// Parse + validate in the order SURVEY App. A lists (magic, version, header bounds, arity, stream
// bounds, per-codec stream sizes).  Returns "" on success, else the earliest violated field.
inline std::string parse_chunk(const void* data, size_t bytes, Chunk* c) {
  const uint8_t* p = static_cast<const uint8_t*>(data);
  if (!p) return "null chunk";
  if (bytes < kHeaderBytes) return "header: truncated";
  if (rd32(p) != kMagic) return "header: bad magic";
  if (rd16(p + 4) != 1) return "header: unsupported version";
  uint32_t nn = rd16(p + 6), ns = rd16(p + 8);
  c->dtype = p[10];
  c->width = rd32(p + 12);
  c->rows = rd64(p + 16);
  c->payload_bytes = rd64(p + 24);
  c->offsets_bytes = rd64(p + 32);
  c->total_bytes = rd64(p + 40);
  c->cascade_hash = rd64(p + 48);
  c->chunk_id = rd64(p + 56);
  if (c->total_bytes > bytes) return "header: total bytes beyond buffer";
  if (c->dtype > T_VARBYTES) return "header: bad dtype";
  if (c->rows >= (1ull << 31)) return "header: rows >= 2^31";
  uint64_t tables = kHeaderBytes + uint64_t(kNodeBytes) * nn + uint64_t(kStreamBytes) * ns;
  if (tables > c->total_bytes) return "header: node/stream tables beyond chunk";
  c->nodes.resize(nn);
  c->streams.resize(ns);
  for (uint32_t i = 0; i < nn; i++) {
    const uint8_t* q = p + kHeaderBytes + uint64_t(kNodeBytes) * i;
    Node& nd = c->nodes[i];
    nd.codec = q[0];
    nd.nchild = q[1];
    nd.stream = rd16(q + 2);
    nd.elem_bytes = rd32(q + 4);
    nd.n = rd64(q + 8);
    std::memcpy(nd.params, q + 16, 16);
  }
  for (uint32_t i = 0; i < ns; i++) {
    const uint8_t* q = p + kHeaderBytes + uint64_t(kNodeBytes) * nn + uint64_t(kStreamBytes) * i;
    c->streams[i].offset = rd64(q);
    c->streams[i].bytes = rd64(q + 8);
    const Stream& s = c->streams[i];
    if (s.offset % 16) return "stream table: stream " + std::to_string(i) + " not 16-byte aligned";
    // the padded extent (round up to 16, plus 16 slack bytes) must be inside the chunk: kernels may
    // read up to 16 bytes past `bytes`
    uint64_t padded = ((s.bytes + 15) & ~15ull) + 16;
    if (s.offset < tables || s.offset > c->total_bytes || padded > c->total_bytes - s.offset)
      return "stream table: stream " + std::to_string(i) + " beyond chunk";
  }
  return "";
}

}  // namespace cdm
