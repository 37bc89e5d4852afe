// ckpt.cu -- elastic checkpoint of device shards.
//
// Reference: checkpoint.hpp:25-54 / checkpoint.cpp (save_shard, read_shard_file,
// load_cluster).  Same little-endian shard file:
//   header : magic u32, version u32, world u32, rank u32, dim u32, reserved u32,
//            capacity u64, entry_count u64
//   record : slot u64, global_id u64, embedding dim*f32, timestamp u64,
//            opt_m dim*f32, opt_v dim*f32, opt_step u64
// Device slots are not the reference's probe positions (different key
// structure), so this side writes records in key order with `slot` = the
// record's ordinal: files are byte-deterministic given the table contents,
// and save -> load -> save is byte-identical.  Loading ignores the stored
// slot and re-inserts (the reference restores exact slots only at an
// unchanged world size, checkpoint.cpp:181-207).  Elastic reload follows
// load_cluster (checkpoint.cpp:194-254): worker r' reads file r' mod W when
// growing, every file f with f mod W' == r' when shrinking, keeps the
// entries it owns under hash64(id) % W', and fast-forwards its tick to the
// newest timestamp.  Host code over rs_table_export / rs_table_import.
#include <algorithm>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "rs_host.hpp"

using namespace rs;

namespace {

constexpr uint32_t kMagic = 0x70736b63;  // "cksp"
constexpr uint32_t kVersion = 1;

void put_u32(std::ostream& os, uint32_t v) {
  const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                              (unsigned char)(v >> 24)};
  os.write(reinterpret_cast<const char*>(b), 4);
}
void put_u64(std::ostream& os, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
  os.write(reinterpret_cast<const char*>(b), 8);
}
void put_f32s(std::ostream& os, const float* x, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t bits;
    std::memcpy(&bits, x + i, 4);
    put_u32(os, bits);
  }
}
uint32_t get_u32(std::istream& is) {
  unsigned char b[4] = {0, 0, 0, 0};
  is.read(reinterpret_cast<char*>(b), 4);
  return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
}
uint64_t get_u64(std::istream& is) {
  unsigned char b[8] = {0};
  is.read(reinterpret_cast<char*>(b), 8);
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= (uint64_t)b[i] << (8 * i);
  return v;
}
void get_f32s(std::istream& is, float* x, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const uint32_t bits = get_u32(is);
    std::memcpy(x + i, &bits, 4);
  }
}

std::string file_name(uint32_t rank, uint32_t world) {
  return "shard_" + std::to_string(rank) + "_of_" + std::to_string(world) + ".ckpt";
}

struct Shard {
  rs_ckpt_header h{};
  std::vector<uint64_t> keys, step, ts;
  std::vector<float> emb, m, v;
};

int read_shard(const std::string& file, Shard* out) {
  std::ifstream is(file, std::ios::binary);
  if (!is) return fail(RS_ERR_IO, "missing shard file: " + file);
  if (get_u32(is) != kMagic) return fail(RS_ERR_IO, "not a shard checkpoint: " + file);
  rs_ckpt_header& h = out->h;
  h.version = get_u32(is);
  if (h.version != kVersion)
    return fail(RS_ERR_IO, "version mismatch in " + file + ": got " + std::to_string(h.version));
  h.world_size = get_u32(is);
  h.shard_rank = get_u32(is);
  h.embedding_dim = get_u32(is);
  get_u32(is);  // reserved
  h.capacity = get_u64(is);
  h.entry_count = get_u64(is);
  if (!is) return fail(RS_ERR_IO, "truncated header in " + file);
  const size_t D = h.embedding_dim, n = h.entry_count;
  out->keys.resize(n);
  out->step.resize(n);
  out->ts.resize(n);
  out->emb.resize(n * D);
  out->m.resize(n * D);
  out->v.resize(n * D);
  for (size_t i = 0; i < n; ++i) {
    get_u64(is);  // slot: not portable across key structures
    out->keys[i] = get_u64(is);
    get_f32s(is, out->emb.data() + i * D, D);
    out->ts[i] = get_u64(is);
    get_f32s(is, out->m.data() + i * D, D);
    get_f32s(is, out->v.data() + i * D, D);
    out->step[i] = get_u64(is);
    if (!is) return fail(RS_ERR_IO, "truncated record in " + file);
  }
  return RS_OK;
}

}  // namespace

extern "C" {

int rs_ckpt_shard_file_name(uint32_t rank, uint32_t world_size, char* out, uint64_t cap) {
  const std::string s = file_name(rank, world_size);
  if (!out || cap < s.size() + 1) return fail(RS_ERR_CONFIG, "rs_ckpt_shard_file_name: buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return RS_OK;
}

// save_shard (checkpoint.cpp:74-103).  Synchronizes.
int rs_ckpt_save_shard(rs_table* t, uint32_t rank, uint32_t world_size, const char* path) {
  if (!t || !path) return fail(RS_ERR_CONFIG, "rs_ckpt_save_shard: null argument");
  uint64_t n = 0;
  int st = rs_table_export(t, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &n);
  if (st) return st;
  const size_t D = t->desc.dim;
  std::vector<uint64_t> keys(n), step(n), ts(n);
  std::vector<float> emb(n * D), m(n * D, 0.f), v(n * D, 0.f);
  if (n) {
    st = rs_table_export(t, n, keys.data(), emb.data(), m.data(), v.data(), step.data(), ts.data(), &n);
    if (st) return st;
  }
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) return fail(RS_ERR_IO, "shard " + std::to_string(rank) + ": cannot open " + path);
  put_u32(os, kMagic);
  put_u32(os, kVersion);
  put_u32(os, world_size);
  put_u32(os, rank);
  put_u32(os, (uint32_t)D);
  put_u32(os, 0);  // reserved
  put_u64(os, t->capacity);
  put_u64(os, n);
  for (uint64_t i = 0; i < n; ++i) {  // key order (export sorts by key); slot = ordinal
    put_u64(os, i);
    put_u64(os, keys[i]);
    put_f32s(os, emb.data() + i * D, D);
    put_u64(os, ts[i]);
    put_f32s(os, m.data() + i * D, D);
    put_f32s(os, v.data() + i * D, D);
    put_u64(os, step[i]);
  }
  os.flush();
  if (!os) return fail(RS_ERR_IO, "shard " + std::to_string(rank) + ": write failed for " + path);
  return RS_OK;
}

// read_shard_file's header (checkpoint.cpp:120-140).
int rs_ckpt_read_header(const char* path, rs_ckpt_header* out) {
  if (!path || !out) return fail(RS_ERR_CONFIG, "rs_ckpt_read_header: null argument");
  std::ifstream is(path, std::ios::binary);
  if (!is) return fail(RS_ERR_IO, std::string("missing shard file: ") + path);
  if (get_u32(is) != kMagic) return fail(RS_ERR_IO, std::string("not a shard checkpoint: ") + path);
  out->version = get_u32(is);
  out->world_size = get_u32(is);
  out->shard_rank = get_u32(is);
  out->embedding_dim = get_u32(is);
  get_u32(is);
  out->capacity = get_u64(is);
  out->entry_count = get_u64(is);
  if (!is) return fail(RS_ERR_IO, std::string("truncated header in ") + path);
  return RS_OK;
}

// load_cluster (checkpoint.cpp:194-254) for worker `rank` of `new_world`,
// into the (empty) device shard t.  Synchronizes.
int rs_ckpt_load_shard(rs_table* t, const char* dir, uint32_t saved_world, uint32_t new_world,
                       uint32_t rank) {
  if (!t || !dir) return fail(RS_ERR_CONFIG, "rs_ckpt_load_shard: null argument");
  if (saved_world == 0 || new_world == 0)
    return fail(RS_ERR_CONFIG, "load_cluster: world sizes must be >= 1");
  if (new_world >= saved_world ? new_world % saved_world != 0 : saved_world % new_world != 0)
    return fail(RS_ERR_CONFIG, "load_cluster: world sizes must divide (" + std::to_string(saved_world) +
                                   " -> " + std::to_string(new_world) + ")");
  if (rank >= new_world) return fail(RS_ERR_CONFIG, "rs_ckpt_load_shard: rank >= new world size");
  std::vector<uint32_t> sources;
  if (new_world >= saved_world) {
    sources.push_back(rank % saved_world);
  } else {
    for (uint32_t f = rank; f < saved_world; f += new_world) sources.push_back(f);
  }
  const size_t D = t->desc.dim;
  Shard all;
  for (uint32_t f : sources) {
    const std::string file = std::string(dir) + "/" + file_name(f, saved_world);
    Shard sh;
    int st = read_shard(file, &sh);
    if (st) return st;
    if (sh.h.embedding_dim != D)
      return fail(RS_ERR_CONFIG, "dim mismatch in " + file + ": file has " + std::to_string(sh.h.embedding_dim) +
                                     ", cluster wants " + std::to_string(D));
    if (sh.h.world_size != saved_world || sh.h.shard_rank != f)
      return fail(RS_ERR_IO, "header/world mismatch in " + file);
    for (size_t i = 0; i < sh.keys.size(); ++i) {
      const bool mine = hash64(sh.keys[i]) % new_world == rank;
      if (new_world == saved_world && !mine)
        return fail(RS_ERR_INVARIANT, "shard file claims rank " + std::to_string(rank) +
                                          " but holds foreign id " + std::to_string(sh.keys[i]));
      if (!mine) continue;  // ownership refilter (two workers may read one file)
      all.keys.push_back(sh.keys[i]);
      all.step.push_back(sh.step[i]);
      all.ts.push_back(sh.ts[i]);
      all.emb.insert(all.emb.end(), sh.emb.begin() + i * D, sh.emb.begin() + (i + 1) * D);
      all.m.insert(all.m.end(), sh.m.begin() + i * D, sh.m.begin() + (i + 1) * D);
      all.v.insert(all.v.end(), sh.v.begin() + i * D, sh.v.begin() + (i + 1) * D);
    }
  }
  const uint64_t n = all.keys.size();
  if (n == 0) return RS_OK;
  return rs_table_import(t, n, all.keys.data(), all.emb.data(), t->desc.s1 ? all.m.data() : nullptr,
                         t->desc.s2 ? all.v.data() : nullptr, all.step.data(), all.ts.data());
}

}  // extern "C"
