// tloom/nn.hpp -- the paper's layer building blocks, executed on the B200 (sm_100a).
//
// Drop-in for the reference operator API (proj/include/tloom/nn.hpp:12-58): identical signatures,
// shape rules and ShapeError messages.  Every call runs a CUDA kernel through the C ABI
// (tlb_nn_* in tloom_b200.h) that evaluates each output element in the reference's summation order, so
// results are bitwise identical to the reference's CPU implementation.
#pragma once

#include "tloom/tensor.hpp"

namespace tloom::nn {

// Output-shape rules; each throws ShapeError on a violated precondition.
Shape conv_result_shape(const Shape& in, const Shape& k);                     // in - k + 1
Shape mconv_result_shape(const Shape& in, const Shape& k, const Shape& b);    // [#k] ++ conv shape
Shape avgpool_result_shape(const Shape& in);                                   // trailing two halved
Shape backavgpool_result_shape(const Shape& in);                               // trailing two doubled
Shape backin_result_shape(const Shape& d_out, const Shape& k, const Shape& in);

Tensor conv(const Tensor& in, const Tensor& k);                    // valid correlation
Tensor mconv(const Tensor& in, const Tensor& k, const Tensor& b);  // stacked biased convolutions
Tensor sigmoid(const Tensor& t);                                   // 1 / (1 + exp(-x))
Tensor backsigmoid(const Tensor& d_out, const Tensor& out);        // d * o * (1 - o)
Tensor avgpool(const Tensor& t);                                   // 2x2 mean, trailing axes
Tensor backavgpool(const Tensor& d_out);                           // adjoint of avgpool
Tensor backweights(const Tensor& d_out, const Tensor& in);         // conv(in, d_out)
float backbias(const Tensor& d_out);                               // sum of the error
Tensor backin(const Tensor& d_out, const Tensor& k, const Tensor& in);  // clipped full correlation

}  // namespace tloom::nn
