// rbd/weight.hpp — WeightSpec (proj/include/rbd/weight.hpp:16-54). The identity
// and diagonal weights run on the B200 path (decompose and the ErrorWorkspace);
// a sparse SPD weight exists only as the external marker of a loaded model.
#ifndef RBD_B200_WEIGHT_HPP
#define RBD_B200_WEIGHT_HPP

#include <cmath>
#include <cstdint>

#include "rbd/errors.hpp"
#include "rbd/types.hpp"

namespace rbd {

enum class WeightKind : std::uint8_t { identity = 0, diagonal = 1, sparse_spd = 2 };

class WeightSpec {
 public:
  WeightSpec() = default;
  static WeightSpec identity() { return WeightSpec(); }
  static WeightSpec diagonal(Vector d) {   // weight.cpp:11-21
    if (d.size() == 0) throw InvalidArgument("diagonal weight must be non-empty");
    for (Index i = 0; i < d.size(); ++i)
      if (!(d[i] > 0.0) || !std::isfinite(d[i]))
        throw InvalidArgument("diagonal weight entries must be strictly positive and finite");
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
