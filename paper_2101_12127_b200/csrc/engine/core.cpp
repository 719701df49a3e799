// core.cpp -- element model and errors (include/dpb200/core.hpp).
#include "dpb200/core.hpp"

#include <sstream>

namespace datapipe::b200 {

const char* ErrorCodeName(ErrorCode code) {
  switch (code) {
    case ErrorCode::kInvalidArity: return "InvalidArity";
    case ErrorCode::kInvalidAttr: return "InvalidAttr";
    case ErrorCode::kTypeMismatch: return "TypeMismatch";
    case ErrorCode::kMalformedInput: return "MalformedInput";
    case ErrorCode::kValidationFailed: return "ValidationFailed";
    case ErrorCode::kDuplicateName: return "DuplicateName";
    case ErrorCode::kUnknownUdf: return "UnknownUdf";
    case ErrorCode::kMissingFile: return "MissingFile";
    case ErrorCode::kUdfError: return "UdfError";
    case ErrorCode::kFingerprintMismatch: return "FingerprintMismatch";
    case ErrorCode::kVersionMismatch: return "VersionMismatch";
    case ErrorCode::kCorruptBlob: return "CorruptBlob";
    case ErrorCode::kConcurrentCacheFill: return "ConcurrentCacheFill";
    case ErrorCode::kRewriteDiverged: return "RewriteDiverged";
    case ErrorCode::kRuleProducedInvalidGraph: return "RuleProducedInvalidGraph";
    case ErrorCode::kDomainError: return "DomainError";
    case ErrorCode::kGridTooLarge: return "GridTooLarge";
    case ErrorCode::kParseError: return "ParseError";
    case ErrorCode::kInternal: return "Internal";
  }
  return "Unknown";
}

size_t DTypeSize(DType t) {
  switch (t) {
    case DType::kUInt8: return 1;
    case DType::kInt32: return 4;
    case DType::kInt64: return 8;
    case DType::kFloat32: return 4;
  }
  return 1;
}

const char* DTypeName(DType t) {
  switch (t) {
    case DType::kUInt8: return "uint8";
    case DType::kInt32: return "int32";
    case DType::kInt64: return "int64";
    case DType::kFloat32: return "float32";
  }
  return "?";
}

int64_t Tensor::num_elements() const {
  int64_t n = 1;
  for (int64_t d : shape) n *= d;
  return n;
}

namespace {
bool SameShapeKind(const Value& a, const Value& b) {
  if (a.kind() != b.kind()) return false;
  if (a.kind() == Value::Kind::kList) {
    if (a.items().empty() || b.items().empty()) return true;
    return SameShapeKind(a.items()[0], b.items()[0]);
  }
  if (a.kind() == Value::Kind::kTuple) {
    if (a.items().size() != b.items().size()) return false;
    for (size_t i = 0; i < a.items().size(); ++i)
      if (!SameShapeKind(a.items()[i], b.items()[i])) return false;
    return true;
  }
  if (a.kind() == Value::Kind::kTensor)
    return a.tensor().dtype == b.tensor().dtype && a.tensor().shape.size() == b.tensor().shape.size();
  return true;
}

std::string ShapeString(const std::vector<int64_t>& shape) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < shape.size(); ++i) os << (i ? "," : "") << (shape[i] < 0 ? std::string("?") : std::to_string(shape[i]));
  os << "]";
  return os.str();
}
}  // namespace

// Homogeneity rule of Value::List (reference element.cpp:21-35): all items
// have the same kind structure; list lengths may differ.
Value Value::List(std::vector<Value> items) {
  for (size_t i = 1; i < items.size(); ++i)
    if (!SameShapeKind(items[0], items[i]))
      throw PipelineError(ErrorCode::kValidationFailed, "list items are not homogeneous");
  return Value(Storage(ListBox{std::move(items)}));
}

const std::vector<Value>& Value::items() const {
  if (kind() == Kind::kList) return std::get<ListBox>(v_).items;
  return std::get<TupleBox>(v_).items;
}

std::string Value::ToString() const {
  std::ostringstream os;
  switch (kind()) {
    case Kind::kInt64: os << int64(); break;
    case Kind::kFloat64: os << float64(); break;
    case Kind::kBytes: os << "b\"" << bytes().size() << " bytes\""; break;
    case Kind::kBool: os << (boolean() ? "true" : "false"); break;
    case Kind::kList:
    case Kind::kTuple: {
      os << (kind() == Kind::kList ? "[" : "(");
      for (size_t i = 0; i < items().size() && i < 8; ++i) os << (i ? ", " : "") << items()[i].ToString();
      if (items().size() > 8) os << ", ...";
      os << (kind() == Kind::kList ? "]" : ")");
      break;
    }
    case Kind::kTensor:
      os << "tensor<" << DTypeName(tensor().dtype) << ShapeString(tensor().shape)
         << (tensor().residency == Residency::kDevice ? "@cuda:" + std::to_string(tensor().device) : "@host") << ">";
      break;
  }
  return os.str();
}

TypeSpec TypeSpec::List(TypeSpec inner, std::optional<uint64_t> length) {
  TypeSpec t(Value::Kind::kList);
  t.nested_.push_back(std::move(inner));
  t.length_ = length;
  return t;
}

TypeSpec TypeSpec::Tuple(std::vector<TypeSpec> members) {
  TypeSpec t(Value::Kind::kTuple);
  t.nested_ = std::move(members);
  return t;
}

TypeSpec TypeSpec::OfTensor(DType dtype, std::vector<int64_t> shape) {
  TypeSpec t(Value::Kind::kTensor);
  t.dtype_ = dtype;
  t.shape_ = std::move(shape);
  return t;
}

bool TypeSpec::Matches(const Value& v) const {
  if (v.kind() != kind_) return false;
  switch (kind_) {
    case Value::Kind::kList:
      if (length_ && v.items().size() != *length_) return false;
      for (const auto& item : v.items())
        if (!nested_[0].Matches(item)) return false;
      return true;
    case Value::Kind::kTuple:
      if (v.items().size() != nested_.size()) return false;
      for (size_t i = 0; i < nested_.size(); ++i)
        if (!nested_[i].Matches(v.items()[i])) return false;
      return true;
    case Value::Kind::kTensor: {
      const Tensor& t = v.tensor();
      if (t.dtype != dtype_ || t.shape.size() != shape_.size()) return false;
      for (size_t i = 0; i < shape_.size(); ++i)
        if (shape_[i] >= 0 && shape_[i] != t.shape[i]) return false;
      return true;
    }
    default:
      return true;
  }
}

bool TypeSpec::operator==(const TypeSpec& o) const {
  return kind_ == o.kind_ && nested_ == o.nested_ && length_ == o.length_ &&
         (kind_ != Value::Kind::kTensor || (dtype_ == o.dtype_ && shape_ == o.shape_));
}

std::string TypeSpec::ToString() const {
  switch (kind_) {
    case Value::Kind::kInt64: return "int64";
    case Value::Kind::kFloat64: return "float64";
    case Value::Kind::kBytes: return "bytes";
    case Value::Kind::kBool: return "bool";
    case Value::Kind::kList:
      return "list<" + nested_[0].ToString() + (length_ ? "," + std::to_string(*length_) : std::string()) + ">";
    case Value::Kind::kTuple: {
      std::string s = "tuple<";
      for (size_t i = 0; i < nested_.size(); ++i) s += (i ? "," : "") + nested_[i].ToString();
      return s + ">";
    }
    case Value::Kind::kTensor:
      return std::string("tensor<") + DTypeName(dtype_) + ShapeString(shape_) + ">";
  }
  return "?";
}

Element::Element(std::vector<Value> components) : components_(std::move(components)) {
  if (components_.empty()) throw PipelineError(ErrorCode::kValidationFailed, "element must have >= 1 component");
}

std::string Element::ToString() const {
  std::string s = "(";
  for (size_t i = 0; i < components_.size(); ++i) s += (i ? ", " : "") + components_[i].ToString();
  return s + ")";
}

std::string ElementSpec::ToString() const {
  std::string s = "(";
  for (size_t i = 0; i < components_.size(); ++i) s += (i ? ", " : "") + components_[i].ToString();
  return s + ")";
}

bool Conforms(const Element& elem, const ElementSpec& spec) {
  if (elem.arity() != spec.arity()) return false;
  for (size_t i = 0; i < spec.arity(); ++i)
    if (!spec.components()[i].Matches(elem.component(i))) return false;
  return true;
}

}  // namespace datapipe::b200
