// dpb200/core.hpp -- element model and errors of the B200 datapipe engine.
//
// Same contracts as the reference's element model (/root/reference/proj/
// include/datapipe/element.hpp:30-184, errors.hpp:25-123), extended with the
// dense tensor value the reference leaves room for ("A dense numeric array
// value MAY be added later behind the same TypeSpec"): batches
// produced by the device path are Elements whose components are Tensors in
// HBM (or pinned host memory), so Conforms is O(1) per component instead of
// the reference's recursive walk over every row.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace datapipe::b200 {

// ---------------------------------------------------------------- errors --
// Values mirror datapipe::ErrorCode (errors.hpp:25-45); the C ABI returns
// code + 1 (include/dpcuda.h).
enum class ErrorCode {
  kInvalidArity,
  kInvalidAttr,
  kTypeMismatch,
  kMalformedInput,
  kValidationFailed,
  kDuplicateName,
  kUnknownUdf,
  kMissingFile,
  kUdfError,
  kFingerprintMismatch,
  kVersionMismatch,
  kCorruptBlob,
  kConcurrentCacheFill,
  kRewriteDiverged,
  kRuleProducedInvalidGraph,
  kDomainError,
  kGridTooLarge,
  kParseError,
  kInternal,
};

const char* ErrorCodeName(ErrorCode code);

class PipelineError : public std::runtime_error {
 public:
  PipelineError(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(ErrorCodeName(code)) + ": " + message), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

// A device-side failure (CUDA error) surfaced through the same hierarchy.
class DeviceError : public PipelineError {
 public:
  explicit DeviceError(const std::string& message) : PipelineError(ErrorCode::kInternal, message) {}
};

// ---------------------------------------------------------------- tensors --
enum class DType : uint8_t { kUInt8 = 0, kInt32 = 1, kInt64 = 2, kFloat32 = 3 };
size_t DTypeSize(DType t);
const char* DTypeName(DType t);

enum class Residency : uint8_t { kDevice = 0, kHost = 1 };

// Dense row-major array.  `owner` keeps the underlying allocation (a ring
// slot lease for iterator outputs) alive for as long as any copy of the
// tensor exists.  `ready` (a cudaEvent_t, may be null) completes when the
// producing kernels have finished writing `data`.
struct Tensor {
  DType dtype = DType::kUInt8;
  std::vector<int64_t> shape;
  void* data = nullptr;
  Residency residency = Residency::kDevice;
  int device = 0;
  std::shared_ptr<void> owner;
  void* ready = nullptr;

  int64_t num_elements() const;
  size_t nbytes() const { return static_cast<size_t>(num_elements()) * DTypeSize(dtype); }
};

// ------------------------------------------------------------------ values --
class Value {
 public:
  enum class Kind : uint8_t { kInt64 = 0, kFloat64 = 1, kBytes = 2, kBool = 3, kList = 4, kTuple = 5, kTensor = 6 };

  static Value Int64(int64_t v) { return Value(Storage(v)); }
  static Value Float64(double v) { return Value(Storage(v)); }
  static Value Bytes(std::string v) { return Value(Storage(BytesBox{std::move(v)})); }
  static Value Bool(bool v) { return Value(Storage(BoolBox{v})); }
  static Value List(std::vector<Value> items);  // homogeneous (kValidationFailed)
  static Value Tuple(std::vector<Value> items) { return Value(Storage(TupleBox{std::move(items)})); }
  static Value FromTensor(Tensor t) { return Value(Storage(std::make_shared<Tensor>(std::move(t)))); }
  static Value FromTensor(std::shared_ptr<Tensor> t) { return Value(Storage(std::move(t))); }

  Kind kind() const { return static_cast<Kind>(v_.index()); }
  int64_t int64() const { return std::get<int64_t>(v_); }
  const int64_t* int64_ptr() const { return &std::get<int64_t>(v_); }  // stable while the Value lives
  double float64() const { return std::get<double>(v_); }
  const std::string& bytes() const { return std::get<BytesBox>(v_).data; }
  bool boolean() const { return std::get<BoolBox>(v_).data; }
  const std::vector<Value>& items() const;
  const Tensor& tensor() const { return *std::get<std::shared_ptr<Tensor>>(v_); }

  std::string ToString() const;

 private:
  struct BytesBox {
    std::string data;
  };
  struct BoolBox {
    bool data;
  };
  struct ListBox {
    std::vector<Value> items;
  };
  struct TupleBox {
    std::vector<Value> items;
  };
  using Storage = std::variant<int64_t, double, BytesBox, BoolBox, ListBox, TupleBox, std::shared_ptr<Tensor>>;
  explicit Value(Storage v) : v_(std::move(v)) {}
  Storage v_;
};

// Static type of a value.  Tensor specs carry the dtype and a shape whose
// unknown dimensions are -1 (e.g. the batch dimension of a partial batch).
class TypeSpec {
 public:
  static TypeSpec Int64() { return TypeSpec(Value::Kind::kInt64); }
  static TypeSpec Float64() { return TypeSpec(Value::Kind::kFloat64); }
  static TypeSpec Bytes() { return TypeSpec(Value::Kind::kBytes); }
  static TypeSpec Bool() { return TypeSpec(Value::Kind::kBool); }
  static TypeSpec List(TypeSpec inner, std::optional<uint64_t> length = std::nullopt);
  static TypeSpec Tuple(std::vector<TypeSpec> members);
  static TypeSpec OfTensor(DType dtype, std::vector<int64_t> shape);

  Value::Kind kind() const { return kind_; }
  const TypeSpec& inner() const { return nested_.at(0); }
  std::optional<uint64_t> length() const { return length_; }
  DType dtype() const { return dtype_; }
  const std::vector<int64_t>& shape() const { return shape_; }

  bool Matches(const Value& v) const;  // O(1) for tensors
  bool operator==(const TypeSpec& o) const;
  bool operator!=(const TypeSpec& o) const { return !(*this == o); }
  std::string ToString() const;

 private:
  explicit TypeSpec(Value::Kind k) : kind_(k) {}
  Value::Kind kind_;
  std::vector<TypeSpec> nested_;
  std::optional<uint64_t> length_;
  DType dtype_ = DType::kUInt8;
  std::vector<int64_t> shape_;
};

class Element {
 public:
  explicit Element(std::vector<Value> components);
  static Element Scalar(Value v) {
    std::vector<Value> c;
    c.push_back(std::move(v));
    return Element(std::move(c));
  }
  const std::vector<Value>& components() const { return components_; }
  size_t arity() const { return components_.size(); }
  const Value& component(size_t i) const { return components_.at(i); }
  std::string ToString() const;

 private:
  std::vector<Value> components_;
};

class ElementSpec {
 public:
  ElementSpec() = default;
  explicit ElementSpec(std::vector<TypeSpec> c) : components_(std::move(c)) {}
  const std::vector<TypeSpec>& components() const { return components_; }
  size_t arity() const { return components_.size(); }
  bool operator==(const ElementSpec& o) const { return components_ == o.components_; }
  bool operator!=(const ElementSpec& o) const { return !(*this == o); }
  std::string ToString() const;

 private:
  std::vector<TypeSpec> components_;
};

bool Conforms(const Element& elem, const ElementSpec& spec);

}  // namespace datapipe::b200
