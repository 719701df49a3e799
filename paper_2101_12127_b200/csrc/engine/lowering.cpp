// lowering.cpp -- Lower(): a graph -> the batch stage, index chain and
// source the device pipeline runs (runtime.cpp has the scheme).
#include <algorithm>
#include <string>

#include "engine/lowering.hpp"

namespace datapipe::b200::detail {
namespace {
[[noreturn]] void Unsupported(const std::string& why) {
  throw PipelineError(ErrorCode::kInvalidAttr, "device lowering: " + why);
}

// A chain of image map steps -> K9's descriptor: the first crop (before any
// resize) is crop A, a crop after the resize -- or a second crop without one
// -- is crop B; pixel ops (normalize, cast = normalize(0, 1), image affine)
// act on the source taps before the resize and on the blend after it.  They
// commute with crops and flips (pointwise, per channel), so only their place
// relative to the resize matters.
dp_image_chain LowerImageChain(const std::vector<MapStep>& steps, int64_t in_h, int64_t in_w) {
  dp_image_chain c{};
  c.in_h = static_cast<int>(in_h);
  c.in_w = static_cast<int>(in_w);
  int ops = 0;
  for (const auto& s : steps) {
    switch (s.op) {
      case MapStep::Op::kRandomCropFlip:
      case MapStep::Op::kCenterCrop: {
        const int mode = s.op == MapStep::Op::kRandomCropFlip ? 1 : 2;
        const bool flip = s.op == MapStep::Op::kRandomCropFlip && s.flip;
        if (!c.resize && !c.pre_mode) {
          c.pre_mode = mode;
          c.pre_h = static_cast<int>(s.out_h);
          c.pre_w = static_cast<int>(s.out_w);
          c.pre_flip = flip;
          c.pre_seed = s.seed;
        } else if (!c.post_mode) {
          c.post_mode = mode;
          c.post_h = static_cast<int>(s.out_h);
          c.post_w = static_cast<int>(s.out_w);
          c.post_flip = flip;
          c.post_seed = s.seed;
        } else {
          Unsupported("image UDF chain: at most one crop before and one after the resize (or two crops)");
        }
        break;
      }
      case MapStep::Op::kResizeBilinear:
        if (c.resize || c.post_mode) Unsupported("image UDF chain: one resize, before any second crop");
        c.resize = 1;
        c.rs_h = static_cast<int>(s.out_h);
        c.rs_w = static_cast<int>(s.out_w);
        break;
      case MapStep::Op::kNormalize:
      case MapStep::Op::kImageAffine: {
        if (ops == 4) Unsupported("image UDF chain: at most 4 pixel ops");
        const bool norm = s.op == MapStep::Op::kNormalize;
        c.op_kind[ops] = norm ? 0 : 1;
        for (int ch = 0; ch < 3; ++ch) {
          c.op_a[ops][ch] = norm ? s.mean[ch] : s.scale[ch];
          c.op_b[ops][ch] = norm ? s.stdv[ch] : s.shift[ch];
        }
        ++ops;
        (c.resize ? c.num_post_ops : c.num_pre_ops)++;
        break;
      }
      default:
        Unsupported("image UDF chain: unsupported map step on images");
    }
  }
  c.out_f32 = c.resize || ops > 0;
  return c;
}

}  // namespace

Lowered Lower(const DatasetGraph& g, const UdfRegistry& reg) {
  Lowered L;
  const DatasetNode* n = g.root().get();
  std::string path = "/" + std::string(NodeKindName(n->kind())) + "@0";
  auto descend = [&]() {
    n = n->inputs()[0].get();
    path += "/" + std::string(NodeKindName(n->kind())) + "@0";
  };
  while (n->kind() == NodeKind::kPrefetch) {
    L.node_paths.push_back(path);
    int64_t b = n->GetInt("buffer_size");
    L.prefetch = (b == kAutotune || L.prefetch == kAutotune) ? kAutotune : std::max(L.prefetch, b);
    descend();
  }
  if (n->kind() == NodeKind::kRepeat) {
    L.node_paths.push_back(path);
    L.outer_repeat = n->GetInt("count");
    descend();
    while (n->kind() == NodeKind::kPrefetch) {
      L.node_paths.push_back(path);
      descend();
    }
  }
  // top-down record of maps and index ops, to give every filter the affine
  // maps beneath it (a value predicate sees mapped values)
  std::vector<IndexOp> top_down;
  struct SeqItem {
    int op;                           // index into top_down, or -1
    const std::vector<MapStep>* map;  // a map's steps
  };
  std::vector<SeqItem> seq;
  auto push_filter = [&](const std::string& udf) {
    const auto& e = reg.Get(udf);
    if (!e.predicate) Unsupported("filter UDF '" + udf + "' is not a device predicate");
    IndexOp op{IndexOp::Kind::kFilter, 0, 0, {}, path};
    op.pred = *e.predicate;
    top_down.push_back(op);
    seq.push_back({static_cast<int>(top_down.size()) - 1, nullptr});
  };
  // ---- batch stage ----
  L.batch_node_path = path;
  L.node_paths.push_back(path);
  if (n->kind() == NodeKind::kMapAndBatch || n->kind() == NodeKind::kBatch) {
    if (n->kind() == NodeKind::kMapAndBatch) L.steps = reg.Get(n->GetString("udf")).map;
    L.batch = n->GetInt("batch_size");
    L.drop = n->GetBoolOr("drop_remainder", false);
    descend();
    // unfused map(f).map(g)...batch: the same result as the fused rewrite for
    // total UDFs (optimizer.cpp map_map / map_batch fusion)
    while (n->kind() == NodeKind::kMap) {
      if (n->HasAttr("fused_filter_udf")) break;  // map(f) + filter: lowered with the index chain
      const auto& f = reg.Get(n->GetString("udf")).map;
      L.steps.insert(L.steps.begin(), f.begin(), f.end());  // inner maps run first
      seq.push_back({-1, &f});
      descend();
    }
  } else if (n->kind() == NodeKind::kPaddedBatch) {
    L.kind = BatchKind::kPadded;
    L.batch = n->GetInt("batch_size");
    L.pad = n->GetInt("padding_value");
    L.drop = n->GetBoolOr("drop_remainder", false);
    descend();
  } else if (n->kind() == NodeKind::kBucketByLength) {
    L.kind = BatchKind::kPadded;
    L.bucketed = true;
    const auto& attrs = n->attrs();
    for (int64_t b : std::get<std::vector<int64_t>>(attrs.at("bucket_boundaries")))
      L.bucket_bounds.push_back(static_cast<int32_t>(b));
    L.bucket_sizes = std::get<std::vector<int64_t>>(attrs.at("bucket_batch_sizes"));
    L.batch = *std::max_element(L.bucket_sizes.begin(), L.bucket_sizes.end());
    L.pad = n->GetInt("padding_value");
    L.drop = n->GetBoolOr("drop_remainder", false);
    descend();
  } else {
    // no batch stage: single elements (the maps under the root run in the
    // internal batch kernels, as under a batch)
    L.unbatched = true;
    L.batch_node_path.clear();
    while (n->kind() == NodeKind::kMap) {
      if (n->HasAttr("fused_filter_udf")) break;
      const auto& f = reg.Get(n->GetString("udf")).map;
      L.steps.insert(L.steps.begin(), f.begin(), f.end());
      seq.push_back({-1, &f});
      descend();
    }
  }
  // ---- index chain ----
  std::vector<MapStep> below;  // maps under the index ops (e.g. from_file.map(decode).shuffle)
  bool seen_interleave = false;
  for (;;) {
    const NodeKind k = n->kind();
    if (k == NodeKind::kShard) {
      top_down.push_back({IndexOp::Kind::kShard, n->GetInt("num_shards"), n->GetInt("index"), {}, path});
    } else if (k == NodeKind::kShuffle) {
      IndexOp op{IndexOp::Kind::kShuffle, n->GetInt("buffer_size"), 0, {}, path};
      if (n->HasAttr("seed")) op.seed = n->GetUint("seed");
      top_down.push_back(op);
    } else if (k == NodeKind::kFilter) {
      push_filter(n->GetString("udf"));
    } else if (k == NodeKind::kRepeat) {
      if (!top_down.empty()) Unsupported("repeat must sit directly under the batch stage");
      top_down.push_back({IndexOp::Kind::kRepeat, n->GetInt("count"), 0, {}, path});
    } else if (k == NodeKind::kInterleave) {
      if (seen_interleave) Unsupported("nested interleave");
      seen_interleave = true;
      const auto& e = reg.Get(n->GetString("udf"));
      if (!e.reader) Unsupported("interleave UDF is not a record reader");
      top_down.push_back({IndexOp::Kind::kInterleave, n->GetInt("cycle_length"), e.reader->records, {}, path,
                          n->GetInt("num_parallel_calls")});
      if (n->HasAttr("records")) L.records = n->GetSource("records");
    } else if (k == NodeKind::kMap) {
      // a map is a pure per-element function whose randomness is keyed by the
      // element id (Philox counter), which travels with the element: it
      // commutes with shard / shuffle / repeat and is run in the batch stage
      // map(f) with a fused predicate (map_filter_fusion) = filter(p) above map(f)
      if (n->HasAttr("fused_filter_udf")) push_filter(n->GetString("fused_filter_udf"));
      if (seen_interleave) Unsupported("map under interleave");
      const auto& f = reg.Get(n->GetString("udf")).map;
      below.insert(below.begin(), f.begin(), f.end());
      seq.push_back({-1, &f});
    } else if (k == NodeKind::kPrefetch) {
      // prefetch inside the index chain only buffers indices: a no-op here
    } else {
      break;
    }
    L.node_paths.push_back(path);
    descend();
  }
  L.node_paths.push_back(path);
  {  // bottom-up: the affine maps beneath each filter
    int64_t mul = 1, add = 0;  // wrap-around int64, as K1
    bool opaque = false;
    for (auto it = seq.rbegin(); it != seq.rend(); ++it) {
      if (it->map) {
        for (const auto& st : *it->map) {
          if (st.op == MapStep::Op::kAffine) {
            mul = static_cast<int64_t>(static_cast<uint64_t>(mul) * static_cast<uint64_t>(st.a));
            add = static_cast<int64_t>(static_cast<uint64_t>(add) * static_cast<uint64_t>(st.a) +
                                       static_cast<uint64_t>(st.b));
          } else {
            opaque = true;
          }
        }
      } else {
        IndexOp& op = top_down[it->op];
        op.mul = mul;
        op.add = add;
        op.opaque = opaque;
      }
    }
  }
  L.chain.assign(top_down.rbegin(), top_down.rend());
  L.steps.insert(L.steps.begin(), below.begin(), below.end());
  // ---- source ----
  switch (n->kind()) {
    case NodeKind::kRange:
      L.source_count = n->GetInt("count");
      break;
    case NodeKind::kFromMemory:
    case NodeKind::kFromFile:
    case NodeKind::kTensorSlices:
    case NodeKind::kTokenSequences:
      L.source = n->GetSource("source");
      L.source_count = L.source->count;
      break;
    default:
      Unsupported(std::string("unsupported node on the device path: ") + NodeKindName(n->kind()));
  }
  if (L.source && L.source->shard_count > 1) {
    // sharded residency: the graph's first transformation must be the shard
    // this process holds; positions then index resident rows directly
    const auto& s = *L.source;
    if (L.chain.empty() || L.chain[0].kind != IndexOp::Kind::kShard || L.chain[0].a != s.shard_count ||
        L.chain[0].b != s.shard_index)
      Unsupported("source holds only shard " + std::to_string(s.shard_index) + " of " +
                  std::to_string(s.shard_count) + ": apply shard(" + std::to_string(s.shard_count) + ", " +
                  std::to_string(s.shard_index) + ") to it first");
    L.chain.erase(L.chain.begin());
    L.source_count = s.count;
  }
  if (seen_interleave) {
    int64_t reader_records = 0;
    for (const auto& op : L.chain)
      if (op.kind == IndexOp::Kind::kInterleave) reader_records = op.b;
    if (L.records && L.records->shard_count > 1) {
      // block residency: this process holds the record files of the
      // interleave inputs shard(k, g) keeps; the interleave then indexes the
      // held files (local file j = input j of the shard)
      const auto& rs = *L.records;
      if (L.chain.size() < 2 || L.chain[0].kind != IndexOp::Kind::kShard || L.chain[0].a != rs.shard_count ||
          L.chain[0].b != rs.shard_index || L.chain[1].kind != IndexOp::Kind::kInterleave)
        Unsupported("records hold only the files of shard " + std::to_string(rs.shard_index) + " of " +
                    std::to_string(rs.shard_count) + ": apply shard(" + std::to_string(rs.shard_count) + ", " +
                    std::to_string(rs.shard_index) + ") to the interleave's inputs, directly");
      if (reader_records != rs.shard_block)
        Unsupported("sharded records hold files of " + std::to_string(rs.shard_block) +
                    " records; the reader opens " + std::to_string(reader_records));
      L.records_local = true;
    }
    if (L.records && !L.source && reader_records > 0) {
      // every record the closed-form interleave names must be resident
      int64_t first = 0, stride = 1, m = L.source_count;
      for (const auto& op : L.chain) {
        if (op.kind != IndexOp::Kind::kShard) break;
        m = m > op.b ? (m - op.b + op.a - 1) / op.a : 0;
        first += op.b * stride;
        stride *= op.a;
      }
      const int64_t need = m == 0 ? 0 : L.records_local ? m * reader_records
                                                         : (first + (m - 1) * stride + 1) * reader_records;
      if (need > L.records->count)
        throw PipelineError(ErrorCode::kMalformedInput,
                            "interleave: the readers open " + std::to_string(need) + " records, the record source holds " +
                                std::to_string(L.records->count));
    }
    if (L.records && L.records->kind == SourceData::Kind::kRecords) {
      // interleave over record files: input element x opens file x.  A
      // reader of R > 0 records requires every file to hold R (records
      // x * R .. x * R + R - 1 of the concatenation, the closed form); a
      // reader of 0 takes each file's own count (unequal files, scheduled).
      int64_t R = 0, p = 1;
      for (const auto& op : L.chain)
        if (op.kind == IndexOp::Kind::kInterleave) {
          R = op.b;
          p = op.parallel;
        }
      bool any_empty = false;
      for (size_t f = 0; f < L.records->file_records.size(); ++f) {
        if (R > 0 && L.records->file_records[f] != R)
          throw PipelineError(ErrorCode::kMalformedInput,
                              "interleave: record file " + std::to_string(f) + " holds " +
                                  std::to_string(L.records->file_records[f]) + " records, the reader opens " +
                                  std::to_string(R) + " (register the reader with 0 records for unequal files)");
        any_empty = any_empty || L.records->file_records[f] == 0;
      }
      // The reference's ParallelInterleaveIterator orders elements around an
      // EMPTY sub-dataset differently from the sequential loop (measured on the
      // compiled reference); only the sequential order is reproduced there.
      if (R == 0 && any_empty && p != 1)
        Unsupported("parallel interleave over record files with an empty file: use num_parallel_calls=1");
    }
    if (L.source && L.source->kind != SourceData::Kind::kInt64) Unsupported("interleave input must be int64 ordinals");
    if (L.source) Unsupported("interleave over from_memory ordinals: use range()");
    L.source = L.records;  // the batch stage reads the record source
    for (const auto& op : L.chain)
      if (op.kind == IndexOp::Kind::kInterleave) break;
      else if (op.kind != IndexOp::Kind::kShard) Unsupported("only shard may precede interleave");
  }
  // ---- from_file records: decode_raw views the packed payloads as images ----
  if (L.source && L.source->kind == SourceData::Kind::kRecords) {
    if (L.steps.empty() || L.steps[0].op != MapStep::Op::kDecodeRaw)
      Unsupported("from_file records must be decoded (decode_raw) before batching");
    const MapStep dec = L.steps[0];
    if (L.source->record_len != dec.out_h * dec.out_w * 3)
      throw PipelineError(ErrorCode::kMalformedInput,
                          "from_file: records are not all " + std::to_string(dec.out_h * dec.out_w * 3) +
                              " bytes (decode_raw " + std::to_string(dec.out_h) + "x" + std::to_string(dec.out_w) +
                              "x3)");
    auto view = std::make_shared<SourceData>(*L.source);
    view->kind = SourceData::Kind::kImages;
    view->h = dec.out_h;
    view->w = dec.out_w;
    view->c = 3;
    L.source = view;
    L.steps.erase(L.steps.begin());
  }
  // ---- batch kind from source + UDF chain ----
  const SourceData::Kind sk = L.source ? L.source->kind : SourceData::Kind::kInt64;
  for (const auto& op : L.chain) {
    if (op.kind != IndexOp::Kind::kFilter) continue;
    if (op.pred.on == DevicePredicate::On::kLength && sk != SourceData::Kind::kTokens)
      Unsupported("a length predicate needs token sequences");
    if (op.pred.on == DevicePredicate::On::kValue && (sk != SourceData::Kind::kInt64 || op.opaque))
      Unsupported("a value predicate needs int64 elements (after affine maps only)");
    if (op.pred.on == DevicePredicate::On::kValue && L.records_local)
      Unsupported("a value predicate over sharded records");
  }
  if (sk == SourceData::Kind::kTokens && L.kind != BatchKind::kPadded) {
    if (!L.steps.empty()) Unsupported("map on token sequences");
    L.kind = BatchKind::kPadded;  // Batch of token sequences (or single ones, internally): ragged
    L.ragged = true;
  }
  if (L.kind == BatchKind::kPadded) {
    if (sk != SourceData::Kind::kTokens) Unsupported("padded_batch needs token sequences");
    for (const auto& op : L.chain)
      if (op.kind == IndexOp::Kind::kRepeat) Unsupported("repeat under padded_batch: put repeat above it");
    if (!L.steps.empty()) Unsupported("map before padded_batch");
  } else if (sk == SourceData::Kind::kInt64) {
    L.kind = BatchKind::kAffine;
    for (const auto& s : L.steps) {
      if (s.op != MapStep::Op::kAffine) Unsupported("int64 elements support affine UDFs only");
      L.affine_a = L.affine_a * s.a;  // (x*a1 + b1)*a2 + b2 in wrap-around int64
      L.affine_b = L.affine_b * s.a + s.b;
    }
  } else {  // images
    const auto& st = L.steps;
    if (st.size() == 2 && st[0].op == MapStep::Op::kRandomCropFlip && st[1].op == MapStep::Op::kNormalize) {
      L.kind = BatchKind::kCrop;
      L.crop = st[0];
      L.norm = st[1];
    } else if (st.size() == 2 && st[0].op == MapStep::Op::kCenterCrop && st[1].op == MapStep::Op::kNormalize) {
      L.kind = BatchKind::kCrop;  // K3 with center offsets
      L.crop = st[0];
      L.norm = st[1];
    } else if (st.size() == 2 && st[0].op == MapStep::Op::kResizeBilinear && st[1].op == MapStep::Op::kNormalize) {
      L.kind = BatchKind::kResize;
      L.resize = st[0];
      L.norm = st[1];
    } else if (st.size() == 1 && st[0].op == MapStep::Op::kResizeBilinear) {
      // resize alone (fp32 out): K4 with the identity normalize, (v - 0) / 1 == v exactly
      L.kind = BatchKind::kResize;
      L.resize = st[0];
      L.norm = MapStep{MapStep::Op::kNormalize};
      L.norm.mean = {0.f, 0.f, 0.f};
      L.norm.stdv = {1.f, 1.f, 1.f};
    } else if (st.size() == 1 && st[0].op == MapStep::Op::kNormalize) {
      // normalize alone: K3 with the whole image as the window (offsets 0, no flip)
      L.kind = BatchKind::kCrop;
      L.crop = MapStep{MapStep::Op::kRandomCropFlip};
      L.crop.out_h = L.source->h;
      L.crop.out_w = L.source->w;
      L.crop.flip = false;
      L.norm = st[0];
    } else if (st.empty()) {
      // Batch with no map: the u8 images themselves (K9 gather)
      L.kind = BatchKind::kCopy;
      L.img_h = L.source->h;
      L.img_w = L.source->w;
    } else {
      L.kind = BatchKind::kChain;
      L.img_chain = LowerImageChain(st, L.source->h, L.source->w);
      int oh = 0, ow = 0, f32 = 0;
      if (dp_image_chain_output(&L.img_chain, &oh, &ow, &f32) != DP_OK)
        Unsupported(std::string("image UDF chain: ") + dp_last_error());
      L.img_h = oh;
      L.img_w = ow;
      L.img_f32 = f32 != 0;
    }
    if (L.source->c != 3) Unsupported("images must have 3 channels");
  }
  // (interleave without a record source emits the int64 record indices
  // themselves: the batch stage gathers them like a range)
  if (L.unbatched) {
    L.batch = L.kind == BatchKind::kAffine || L.kind == BatchKind::kIdentityInt ? 4096
              : L.ragged                                                         ? 1024
                                                                                 : 64;  // internal unit
    L.drop = false;
  }
  return L;
}

}  // namespace datapipe::b200::detail
