// PyTorch operator library of the B200 engine: torch.ops.b2conv.conv2d /
// conv2d_out (BASELINE.json north star: "exposed as a PyTorch C++
// extension").
//
// A thin adapter over the C ABI (include/b2conv.h): it validates the tensors,
// builds the descriptor, takes scratch memory from torch's caching allocator
// on the current stream (so concurrent streams never share a workspace) and
// launches through b2c_conv2d_forward / _tc / b2c_conv_twostage on
// c10::cuda::getCurrentCUDAStream().  The kernels live in libb2conv.so, which
// has no torch dependency; this translation unit is the only one that sees
// torch headers.  A Meta kernel gives shapes to fake-tensor tracing
// (torch.compile, torch.export) without touching the device.
//
// Replaces, for CUDA tensors, the entry point
// convkit.twostage.conv_twostage(inp, filters, cfg) (twostage.py:208-212)
// with F.conv2d's (stride, padding) arguments.
#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include <string>

#include "../../include/b2conv.h"

namespace {

int32_t engine_id(const std::string &e) {
  if (e == "fused") return B2C_ENGINE_FUSED;
  if (e == "twostage") return B2C_ENGINE_TWOSTAGE;
  if (e == "tf32x3") return B2C_ENGINE_TF32X3;
  if (e == "tf32") return B2C_ENGINE_TF32;
  TORCH_CHECK(false, "b2conv: unknown engine '", e, "' (fused, twostage, tf32x3, tf32)");
  return -1;
}

void check_status(b2c_status st, const char *what) {
  TORCH_CHECK(st == B2C_OK, "b2conv.", what, " failed (status ", static_cast<int>(st), "): ", b2c_last_error());
}

b2c_conv_desc make_desc(const at::Tensor &x, const at::Tensor &w, at::IntArrayRef stride, at::IntArrayRef padding) {
  TORCH_CHECK(x.dim() == 4 && w.dim() == 4, "b2conv.conv2d: expected 4-D NCHW input and MCHW filters, got ",
              x.sizes(), " / ", w.sizes());
  TORCH_CHECK(stride.size() == 2 && padding.size() == 2, "b2conv.conv2d: stride and padding are pairs");
  TORCH_CHECK(stride[0] == stride[1], "b2conv.conv2d: one stride for both axes (configs.py:26), got ", stride);
  TORCH_CHECK(w.size(1) == x.size(1), "b2conv.conv2d: filter depth ", w.size(1), " != input channels ", x.size(1));
  b2c_conv_desc d;
  d.n = static_cast<int32_t>(x.size(0));
  d.c = static_cast<int32_t>(x.size(1));
  d.h = static_cast<int32_t>(x.size(2));
  d.w = static_cast<int32_t>(x.size(3));
  d.m = static_cast<int32_t>(w.size(0));
  d.hf = static_cast<int32_t>(w.size(2));
  d.wf = static_cast<int32_t>(w.size(3));
  d.stride = static_cast<int32_t>(stride[0]);
  d.pad_h = static_cast<int32_t>(padding[0]);
  d.pad_w = static_cast<int32_t>(padding[1]);
  return d;
}

std::vector<int64_t> out_shape(const b2c_conv_desc &d) {
  int32_t ho = 0, wo = 0;
  check_status(b2c_output_dims(&d, &ho, &wo), "conv2d");
  return {d.n, d.m, ho, wo};
}

void check_cuda_f32(const at::Tensor &t, const char *what, const at::Device &dev) {
  TORCH_CHECK(t.is_cuda(), "b2conv.conv2d: ", what, " must be a CUDA tensor (the B200 engine has no CPU path)");
  TORCH_CHECK(t.scalar_type() == at::kFloat, "b2conv.conv2d: ", what, " must be float32, got ", t.scalar_type());
  TORCH_CHECK(t.is_contiguous(), "b2conv.conv2d: ", what, " must be contiguous NCHW");
  TORCH_CHECK(t.device() == dev, "b2conv.conv2d: ", what, " is on ", t.device(), ", input on ", dev);
}

at::Tensor &conv2d_out_cuda(const at::Tensor &x, const at::Tensor &w, at::IntArrayRef stride, at::IntArrayRef padding,
                            c10::string_view engine, at::Tensor &out) {
  const b2c_conv_desc d = make_desc(x, w, stride, padding);
  check_cuda_f32(x, "input", x.device());
  check_cuda_f32(w, "filters", x.device());
  check_cuda_f32(out, "out", x.device());
  TORCH_CHECK(out.sizes() == at::IntArrayRef(out_shape(d)), "b2conv.conv2d: out has shape ", out.sizes(),
              ", expected ", at::IntArrayRef(out_shape(d)));
  const int32_t eng = engine_id(std::string(engine));
  c10::cuda::CUDAGuard guard(x.device());
  cudaStream_t stream = c10::cuda::getCurrentCUDAStream(x.device().index()).stream();
  const auto bytes = x.options().dtype(at::kByte);
  const float *xp = x.const_data_ptr<float>();
  const float *wp = w.const_data_ptr<float>();
  float *yp = out.mutable_data_ptr<float>();
  if (eng == B2C_ENGINE_FUSED) {
    b2c_tile_plan tp{};
    tp.family = -1;
    check_status(b2c_select_tiles(&d, eng, &tp), "select_tiles");
    at::Tensor ws;  // split-C partial planes, from the caching allocator on this stream
    if (tp.workspace_bytes > 0) ws = at::empty({tp.workspace_bytes}, bytes);
    check_status(b2c_conv2d_forward(&d, xp, wp, yp, tp.workspace_bytes > 0 ? ws.data_ptr() : nullptr,
                                    tp.workspace_bytes, nullptr, stream),
                 "conv2d");
  } else if (eng == B2C_ENGINE_TWOSTAGE) {
    const int64_t need = b2c_workspace_bytes(&d);
    at::Tensor ws;
    if (need > 0) ws = at::empty({need}, bytes);
    b2c_run_stats stats{};
    check_status(b2c_conv_twostage(&d, xp, wp, yp, need > 0 ? static_cast<float *>(ws.data_ptr()) : nullptr, need,
                                   nullptr, nullptr, INT64_MAX, stream, &stats),
                 "conv_twostage");
  } else {
    b2c_tc_plan tp{};
    check_status(b2c_tc_select_tiles(&d, eng, &tp), "tc_select_tiles");
    at::Tensor ws = at::empty({tp.workspace_bytes > 0 ? tp.workspace_bytes : 16}, bytes);
    check_status(b2c_conv2d_forward_tc(&d, xp, wp, yp, ws.data_ptr(), tp.workspace_bytes, eng, nullptr, stream),
                 "conv2d_tc");
  }
  return out;
}

at::Tensor conv2d_cuda(const at::Tensor &x, const at::Tensor &w, at::IntArrayRef stride, at::IntArrayRef padding,
                       c10::string_view engine) {
  const b2c_conv_desc d = make_desc(x, w, stride, padding);
  at::Tensor out = at::empty(out_shape(d), x.options());
  conv2d_out_cuda(x, w, stride, padding, engine, out);
  return out;
}

at::Tensor conv2d_meta(const at::Tensor &x, const at::Tensor &w, at::IntArrayRef stride, at::IntArrayRef padding,
                       c10::string_view engine) {
  (void)engine_id(std::string(engine));
  const b2c_conv_desc d = make_desc(x, w, stride, padding);
  TORCH_CHECK(x.scalar_type() == at::kFloat && w.scalar_type() == at::kFloat, "b2conv.conv2d: float32 operands");
  return at::empty(out_shape(d), x.options());
}

at::Tensor &conv2d_out_meta(const at::Tensor &x, const at::Tensor &w, at::IntArrayRef stride,
                            at::IntArrayRef padding, c10::string_view engine, at::Tensor &out) {
  (void)engine_id(std::string(engine));
  const b2c_conv_desc d = make_desc(x, w, stride, padding);
  TORCH_CHECK(out.sizes() == at::IntArrayRef(out_shape(d)), "b2conv.conv2d: out has shape ", out.sizes());
  return out;
}

}  // namespace

TORCH_LIBRARY(b2conv, m) {
  m.def("conv2d(Tensor x, Tensor w, int[2] stride=1, int[2] padding=0, str engine='fused') -> Tensor");
  m.def("conv2d_out(Tensor x, Tensor w, int[2] stride, int[2] padding, str engine, *, Tensor(a!) out) -> Tensor(a!)");
}

TORCH_LIBRARY_IMPL(b2conv, CUDA, m) {
  m.impl("conv2d", &conv2d_cuda);
  m.impl("conv2d_out", &conv2d_out_cuda);
}

TORCH_LIBRARY_IMPL(b2conv, Meta, m) {
  m.impl("conv2d", &conv2d_meta);
  m.impl("conv2d_out", &conv2d_out_meta);
}
