// TORCH_LIBRARY(ubs, m): the C ABI of libubs_b200.so (include/ubs_b200.h) as
// PyTorch operators, so torch code (and torch.autograd, via
// paper_2510_03312_b200/ops.py) calls the sm_100a render path on tensors:
//
//   ubs::scene_statics   query-invariant half of slice_scene (slicing.py:185-235)
//   ubs::render          one frame: slice + project + order + build_tiles +
//                        tile_forward over all tiles (raster.py:269-316)
//   ubs::render_backward the frame's parameter gradient for a given dL/dimage
//                        (gradients.py:130-300: tile_backward, scatter, chain)
//   ubs::loss_image_grad L1 + SSIM image gradient (gradients.py:110-116, metrics.py:74-114)
//   ubs::adam_step_      Adam + shape clamp on the packed records (optim.py:115-135)
//
// Host C++ over the same extern "C" entry points the ctypes engine uses; all
// buffers are torch allocations on the current CUDA stream.  render reads
// the tile-pair count K back once (16 bytes) to size the pair buffers, and
// re-runs with a doubled list cap if a capped tile list ran out (the
// engine's synchronous frame, engine.render_frame).
#include <ATen/cuda/CUDAContext.h>
#include <torch/library.h>
#include <torch/torch.h>

#include <cmath>
#include <vector>

#include "ubs_b200.h"

namespace {

constexpr int kTile = 16;
constexpr int kChunkRanks = 1024;  // csrc/binning.cu kCtaRanks
constexpr int kBand = 8, kRows = 4;

void check(int rc, const char *what) {
    TORCH_CHECK(rc == UBS_OK, what, " failed (", rc == UBS_E_ARGS ? "bad arguments" : rc == UBS_E_CUDA ? "CUDA error"
                                                                                     : "capacity", ")");
}

int record_width(int64_t n_dims) { return 14 + 6 * ((int)n_dims - 3); }

void* ptr(const at::Tensor &t) { return t.defined() ? t.data_ptr() : nullptr; }

// camera: f64 [fx, fy, cx, cy, world_to_cam[:3,:3] (9, row-major), world_to_cam[:3,3] (3), width, height]
// settings: f64 [tau_sq, alpha_clamp, transmittance_min, near_plane, cull_margin, screen_cov_floor,
//                psd_floor_scale, gate_symmetric, tile_size]
UbsView make_view(const at::Tensor &params, int64_t n_dims, const at::Tensor &camera, const at::Tensor &query,
                  const at::Tensor &settings, const at::Tensor &background, const at::Tensor &statics) {
    TORCH_CHECK(params.is_cuda() && params.dim() == 2 && params.size(1) == record_width(n_dims) &&
                    params.is_contiguous(), "params must be a contiguous CUDA (n, 14+6C) tensor");
    TORCH_CHECK(params.scalar_type() == at::kFloat || params.scalar_type() == at::kDouble, "params f32 or f64");
    const auto cam = camera.to(at::kCPU, at::kDouble).contiguous();
    const auto q = query.to(at::kCPU, at::kDouble).contiguous();
    const auto st = settings.to(at::kCPU, at::kDouble).contiguous();
    const auto bg = background.to(at::kCPU, at::kDouble).contiguous();
    TORCH_CHECK(cam.numel() == 18 && st.numel() == 9 && bg.numel() == 3, "camera[18], settings[9], background[3]");
    const int c = (int)n_dims - 3;
    TORCH_CHECK(q.numel() == c, "query has ", q.numel(), " dims, scene expects ", c);
    const double *cp = cam.data_ptr<double>(), *sp = st.data_ptr<double>();
    UbsView v{};
    v.params = params.data_ptr();
    v.n = params.size(0);
    v.n_dims = (int32_t)n_dims;
    v.param_f64 = params.scalar_type() == at::kDouble;
    for (int k = 0; k < 3; ++k) v.background[k] = bg.data_ptr<double>()[k];
    for (int k = 0; k < 4; ++k) v.query[k] = k < c ? q.data_ptr<double>()[k] : 0.0;
    v.cam.fx = cp[0]; v.cam.fy = cp[1]; v.cam.cx = cp[2]; v.cam.cy = cp[3];
    for (int k = 0; k < 9; ++k) v.cam.rot[k] = cp[4 + k];
    for (int k = 0; k < 3; ++k) v.cam.trans[k] = cp[13 + k];
    v.cam.width = (int32_t)cp[16];
    v.cam.height = (int32_t)cp[17];
    v.set.tau_sq = sp[0]; v.set.alpha_clamp = sp[1]; v.set.transmittance_min = sp[2];
    v.set.near_plane = sp[3]; v.set.cull_margin = sp[4]; v.set.screen_cov_floor = sp[5];
    v.set.psd_floor_scale = sp[6]; v.set.gate_symmetric = sp[7] != 0.0; v.set.tile_size = (int32_t)sp[8];
    TORCH_CHECK(v.set.tile_size == kTile, "tile_size must be 16");
    v.statics = statics.defined() ? statics.data_ptr() : nullptr;
    return v;
}

at::Tensor scene_statics(const at::Tensor &params, int64_t n_dims, double psd_floor_scale) {
    TORCH_CHECK(params.is_cuda() && params.dim() == 2 && params.size(1) == record_width(n_dims), "params");
    const int f64 = params.scalar_type() == at::kDouble;
    const auto p = params.contiguous();
    auto out = at::empty({(int64_t)ubs_statics_bytes(p.size(0), (int32_t)n_dims, f64)}, p.options().dtype(at::kByte));
    UbsView v{};
    v.params = p.data_ptr();
    v.n = p.size(0);
    v.n_dims = (int32_t)n_dims;
    v.param_f64 = f64;
    v.set.psd_floor_scale = psd_floor_scale;
    check(ubs_scene_statics(&v, out.data_ptr(), at::cuda::getCurrentCUDAStream().stream()), "ubs_scene_statics");
    return out;
}

// Every buffer of one frame (engine.Workspace), torch-allocated.
struct Frame {
    at::Tensor depth_key, rect, tile_count, flags, rec32, rec64, counters, tile_grid, keys_sorted, rect_sorted,
        ids_iota, order, hit_clamp, image, asum, tstop, ncontrib, fix_list, chunk_hist, seg_scratch, bucket_start,
        status, tile_ranges, temp, tile_ids, entries;
    UbsPrimBuffers pb{};
    UbsBinBuffers bb{};
    UbsImageBuffers ib{};
    bool f64 = false;
};

void render_into(Frame &f, const UbsView &v, bool f64, cudaStream_t s) {
    const auto dev = at::TensorOptions().device(at::kCUDA, at::cuda::current_device());
    const int64_t n = std::max<int64_t>(v.n, 1);
    const int W = v.cam.width, H = v.cam.height;
    const int TX = (W + kTile - 1) / kTile, TY = (H + kTile - 1) / kTile;
    const int64_t npix = (int64_t)W * H, ntiles = (int64_t)TX * TY;
    const int64_t nbk = (int64_t)((TY + kRows - 1) / kRows) * ((TX + kBand - 1) / kBand);
    const int64_t G = std::max<int64_t>(1, (v.n + kChunkRanks - 1) / kChunkRanks);
    const auto i64 = dev.dtype(at::kLong), i32 = dev.dtype(at::kInt), fdt = dev.dtype(f64 ? at::kDouble : at::kFloat);
    f.f64 = f64;
    f.depth_key = at::empty({n}, i64);
    f.rect = at::empty({n}, i64);
    f.tile_count = at::empty({n}, i32);
    f.flags = at::empty({n}, dev.dtype(at::kShort));
    f.rec64 = at::empty({n * 10}, dev.dtype(at::kDouble));
    if (!f64) f.rec32 = at::empty({n * 16}, dev.dtype(at::kFloat));
    f.counters = at::zeros({8}, i64);
    f.tile_grid = at::empty({(int64_t)(TX + 1) * (TY + 1)}, i32);
    f.keys_sorted = at::empty({n}, i64);
    f.rect_sorted = at::empty({n}, i64);
    f.ids_iota = at::empty({n}, i32);
    f.order = at::empty({n}, i32);
    f.hit_clamp = at::zeros({n}, dev.dtype(at::kByte));
    f.image = at::empty({H, W, 3}, fdt);
    f.asum = at::empty({H, W}, fdt);
    f.tstop = at::empty({H, W}, fdt);
    f.ncontrib = at::empty({H, W}, i32);
    f.fix_list = at::empty({std::max<int64_t>(npix, 1)}, i32);
    f.chunk_hist = at::empty({10 * G * nbk}, i32);
    f.seg_scratch = at::empty({nbk + 1}, i32);
    f.bucket_start = at::empty({nbk + 1}, i32);
    f.status = at::zeros({1}, i32);
    f.tile_ranges = at::empty({2 * ntiles}, i32);
    f.temp = at::empty({(int64_t)ubs_bin_temp_bytes(v.n, 0, (int32_t)ntiles) + 1}, dev.dtype(at::kByte));
    char *cnt = (char *)f.counters.data_ptr();
    UbsPrimBuffers &pb = f.pb;
    pb.depth_key = (uint64_t *)ptr(f.depth_key);
    pb.rect = (uint64_t *)ptr(f.rect);
    pb.tile_count = (uint32_t *)ptr(f.tile_count);
    pb.flags = (uint16_t *)ptr(f.flags);
    pb.rec32 = f64 ? nullptr : ptr(f.rec32);
    pb.rec64 = ptr(f.rec64);
    pb.n_visible = (uint32_t *)(cnt + 16);
    pb.n_pairs = (unsigned long long *)cnt;
    pb.tile_grid = (int32_t *)ptr(f.tile_grid);
    pb.depth_range = (unsigned long long *)(cnt + 40);
    check(ubs_preprocess(&v, &pb, f64 ? 0 : 1, s), "ubs_preprocess");
    UbsBinBuffers &bb = f.bb;
    bb.keys_sorted = (uint64_t *)ptr(f.keys_sorted);
    bb.rect_sorted = (uint64_t *)ptr(f.rect_sorted);
    bb.ids_iota = (uint32_t *)ptr(f.ids_iota);
    bb.order = (uint32_t *)ptr(f.order);
    bb.tile_ranges = (uint32_t *)ptr(f.tile_ranges);
    bb.temp = ptr(f.temp);
    bb.temp_bytes = (size_t)f.temp.numel();
    bb.chunk_hist = (uint32_t *)ptr(f.chunk_hist);
    bb.chunk_hist_capacity = f.chunk_hist.numel();
    bb.chunk_count = (int32_t)G;
    bb.seg_scratch = (uint32_t *)ptr(f.seg_scratch);
    bb.bucket_start = (uint32_t *)ptr(f.bucket_start);
    bb.bucket_capacity = f.bucket_start.numel();
    bb.status = (uint32_t *)ptr(f.status);
    check(ubs_bin_depth(&v, &pb, &bb, s), "ubs_bin_depth");
    const int64_t K = f.counters.slice(0, 0, 1).cpu().item<int64_t>();  // the frame's one readback
    TORCH_CHECK(K < ((int64_t)1 << 32), K, " tile pairs exceed the 2^32 device limit");
    f.tile_ids = at::empty({std::max<int64_t>(K, 1)}, i32);
    f.entries = at::empty({std::max<int64_t>(K, 1)}, i64);
    bb.tile_ids = (uint32_t *)ptr(f.tile_ids);
    bb.entries = (uint64_t *)ptr(f.entries);
    bb.pair_capacity = std::max<int64_t>(K, 1);
    UbsImageBuffers &ib = f.ib;
    ib.image = ptr(f.image);
    ib.alpha_sum = ptr(f.asum);
    ib.t_stop = ptr(f.tstop);
    ib.n_contrib = (int32_t *)ptr(f.ncontrib);
    ib.hit_clamp = (uint8_t *)ptr(f.hit_clamp);
    ib.visits = (unsigned long long *)(cnt + 8);
    ib.fix_list = (uint32_t *)ptr(f.fix_list);
    ib.fix_count = (uint32_t *)(cnt + 24);
    ib.raster_f64 = f64;
    for (uint32_t cap = 1024;; cap *= 2) {
        bb.list_cap = cap >= (1u << 30) ? 0xFFFFFFFFu : cap;
        check(ubs_bin_tiles(&v, &pb, &bb, K, s), "ubs_bin_tiles");
        check(ubs_raster_forward(&v, &pb, &bb, &ib, s), "ubs_raster_forward");
        check(ubs_raster_fixup(&v, &pb, &bb, &ib, s), "ubs_raster_fixup");
        if (bb.list_cap == 0xFFFFFFFFu || (f.status.cpu().item<int>() & UBS_S_LIST_TRUNC) == 0) break;
        f.status.zero_();  // a capped list ran out: redo the lists and the composite with the cap doubled
        f.hit_clamp.zero_();
        f.counters.slice(0, 1, 2).zero_();  // visits
        f.counters.slice(0, 3, 4).zero_();  // fix count
    }
}

std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor, at::Tensor> render(
    const at::Tensor &params, int64_t n_dims, const at::Tensor &camera, const at::Tensor &query,
    const at::Tensor &settings, const at::Tensor &background, const std::optional<at::Tensor> &statics, bool fp64) {
    const at::Tensor st = statics.has_value() ? *statics : at::Tensor();
    const UbsView v = make_view(params.contiguous(), n_dims, camera, query, settings, background, st);
    Frame f;
    render_into(f, v, fp64, at::cuda::getCurrentCUDAStream().stream());
    return {f.image, f.asum, f.tstop, f.ncontrib, f.hit_clamp.narrow(0, 0, params.size(0)).to(at::kBool)};
}

at::Tensor render_backward(const at::Tensor &params_in, int64_t n_dims, const at::Tensor &camera,
                           const at::Tensor &query, const at::Tensor &settings, const at::Tensor &background,
                           const at::Tensor &g_image, bool fp64) {
    const auto params = params_in.contiguous();
    const UbsView v = make_view(params, n_dims, camera, query, settings, background, at::Tensor());
    cudaStream_t s = at::cuda::getCurrentCUDAStream().stream();
    Frame f;
    render_into(f, v, fp64, s);
    const int64_t n = std::max<int64_t>(params.size(0), 1);
    const auto gdt = fp64 ? at::kDouble : at::kFloat;
    auto gimg = g_image.to(params.device(), gdt).contiguous();
    TORCH_CHECK(gimg.numel() == f.image.numel(), "g_image must match the image shape");
    auto grad2d = at::zeros({n * 12}, params.options().dtype(gdt));
    auto grads = at::zeros_like(params, params.options().dtype(at::kDouble));
    auto nonfinite = at::zeros({1}, params.options().dtype(at::kInt));
    auto active = at::empty({n}, params.options().dtype(at::kInt));
    auto active_count = at::zeros({1}, params.options().dtype(at::kInt));
    UbsGradBuffers gb{};
    gb.g_image = gimg.data_ptr();
    gb.grad2d = grad2d.data_ptr();
    gb.grad_params = grads.data_ptr();
    gb.grad_f64 = 1;
    gb.grad2d_f64 = fp64;
    gb.nonfinite = (uint32_t *)nonfinite.data_ptr();
    gb.flags = f.pb.flags;
    gb.active = (uint32_t *)active.data_ptr();
    gb.active_count = (uint32_t *)active_count.data_ptr();
    gb.bwd_pixels_per_lane = 4;
    if (params.size(0) > 0) {
        check(ubs_raster_backward(&v, &f.pb, &f.bb, &f.ib, &gb, s), "ubs_raster_backward");
        check(ubs_prim_backward(&v, &gb, 0, s), "ubs_prim_backward");
    }
    return grads.to(params.scalar_type());
}

std::tuple<at::Tensor, at::Tensor> loss_image_grad(const at::Tensor &image, const at::Tensor &target,
                                                   double lambda_ssim, double scale) {
    TORCH_CHECK(image.is_cuda() && image.dim() == 3 && image.size(2) == 3, "image must be a CUDA (H, W, 3) tensor");
    const int f64 = image.scalar_type() == at::kDouble;
    const auto a = image.contiguous();
    const auto b = target.to(a.device(), a.scalar_type()).contiguous();
    TORCH_CHECK(b.sizes() == a.sizes(), "target shape");
    const int H = (int)a.size(0), W = (int)a.size(1);
    auto g = at::empty_like(a);
    auto parts = at::zeros({2}, a.options().dtype(at::kDouble));
    auto scratch = at::empty({(int64_t)ubs_loss_scratch_bytes(H, W, f64)}, a.options().dtype(at::kByte));
    check(ubs_loss_image_grad(a.data_ptr(), b.data_ptr(), H, W, f64, lambda_ssim, scale, g.data_ptr(),
                              parts.data_ptr<double>(), scratch.data_ptr(), at::cuda::getCurrentCUDAStream().stream()),
          "ubs_loss_image_grad");
    return {g, parts};
}

void adam_step_(at::Tensor params, const at::Tensor &grads, at::Tensor m, at::Tensor v, int64_t n_dims,
                at::ArrayRef<double> lr, int64_t step, bool freeze_shapes) {
    TORCH_CHECK(lr.size() == 4, "lr = (position, opacity, scale, other)");
    TORCH_CHECK(params.is_contiguous() && grads.is_contiguous() && m.is_contiguous() && v.is_contiguous(),
                "contiguous tensors");
    TORCH_CHECK(m.scalar_type() == at::kFloat && v.scalar_type() == at::kFloat, "f32 moments");
    check(ubs_adam_step(params.data_ptr(), params.scalar_type() == at::kDouble, grads.data_ptr(),
                        grads.scalar_type() == at::kDouble, m.data_ptr<float>(), v.data_ptr<float>(), params.size(0),
                        (int32_t)n_dims, lr.data(), (int32_t)step, freeze_shapes, at::cuda::getCurrentCUDAStream().stream()),
          "ubs_adam_step");
}

}  // namespace

TORCH_LIBRARY(ubs, m) {
    m.def("scene_statics(Tensor params, int n_dims, float psd_floor_scale) -> Tensor");
    m.def("render(Tensor params, int n_dims, Tensor camera, Tensor query, Tensor settings, Tensor background, "
          "Tensor? statics=None, bool fp64=False) -> (Tensor image, Tensor alpha_sum, Tensor t_stop, "
          "Tensor n_contrib, Tensor alpha_clamped)");
    m.def("render_backward(Tensor params, int n_dims, Tensor camera, Tensor query, Tensor settings, "
          "Tensor background, Tensor g_image, bool fp64=False) -> Tensor");
    m.def("loss_image_grad(Tensor image, Tensor target, float lambda_ssim, float scale) -> (Tensor, Tensor)");
    m.def("adam_step_(Tensor(a!) params, Tensor grads, Tensor(b!) m, Tensor(c!) v, int n_dims, float[] lr, "
          "int step, bool freeze_shapes=False) -> ()");
}

TORCH_LIBRARY_IMPL(ubs, CUDA, m) {
    m.impl("scene_statics", &scene_statics);
    m.impl("render", &render);
    m.impl("render_backward", &render_backward);
    m.impl("loss_image_grad", &loss_image_grad);
    m.impl("adam_step_", &adam_step_);
}
