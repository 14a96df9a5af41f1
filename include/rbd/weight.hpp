// rbd/weight.hpp — WeightSpec (proj/include/rbd/weight.hpp:16-54). Only the
// identity weight runs on the B200 path; a diagonal weight is carried for the
// reference's dimension check (IncompatibleWeight) and is otherwise rejected
// with InvalidArgument (next row).
#ifndef RBD_B200_WEIGHT_HPP
#define RBD_B200_WEIGHT_HPP

#include <cstdint>

#include "rbd/types.hpp"

namespace rbd {

enum class WeightKind : std::uint8_t { identity = 0, diagonal = 1, sparse_spd = 2 };

class WeightSpec {
 public:
  WeightSpec() = default;
  static WeightSpec identity() { return WeightSpec(); }
  static WeightSpec diagonal(Vector d) {
    WeightSpec w;
    w.kind_ = WeightKind::diagonal;
    w.diag_ = std::move(d);
    return w;
  }
  // marker for a model whose sparse SPD weight lives outside the model file
  // (weight.hpp:26-28); carries the kind only
  static WeightSpec sparse_external() {
    WeightSpec w;
    w.kind_ = WeightKind::sparse_spd;
    w.external_ = true;
    return w;
  }
  WeightKind kind() const { return kind_; }
  Index dim() const { return kind_ == WeightKind::diagonal ? diag_.size() : 0; }
  bool compatible_with(Index m) const {
    return kind_ == WeightKind::identity || external_ || dim() == m;
  }
  bool evaluable() const { return !external_; }
  const Vector& diagonal_values() const { return diag_; }

 private:
  WeightKind kind_ = WeightKind::identity;
  Vector diag_;
  bool external_ = false;
};

}  // namespace rbd

#endif
