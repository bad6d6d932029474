// PyTorch-facing allocator hooks for liblms (the binding layer, not the pool).
//
// CUDAPluggableAllocator's alloc_fn has no error channel.  Throwing
// c10::OutOfMemoryError here makes an exhausted budget look exactly like a
// CUDA OOM to PyTorch: Python sees torch.OutOfMemoryError, and cuDNN's plan
// loop (which catches c10::OutOfMemoryError) falls back to plans that need a
// smaller workspace instead of failing the step.
#include <c10/util/Exception.h>
#include <cuda_runtime.h>
#include <torch/csrc/cuda/CUDAPluggableAllocator.h>

#include "../../include/lms.h"

extern "C" void* lms_torch_alloc(size_t size, int device, cudaStream_t stream) {
  (void)device;
  lms_ctx* c = lms_get_global();
  TORCH_CHECK(c != nullptr, "LMS: allocator hook used before lms_set_global");
  void* p = nullptr;
  int rc = lms_dev_alloc(c, size, stream, &p);
  if (rc == LMS_E_OOM) {
    TORCH_CHECK_WITH(OutOfMemoryError, false, lms_last_error());
  }
  TORCH_CHECK(rc == LMS_OK, "LMS allocation failed: ", lms_last_error());
  return p;
}

extern "C" void lms_torch_free(void* ptr, size_t size, int device, cudaStream_t stream) {
  (void)size;
  (void)device;
  lms_ctx* c = lms_get_global();
  if (c) lms_dev_free(c, ptr, stream);
}

// Tensor.record_stream(s) on a block of ours: hold its reuse for `s`'s work
// (ProcessGroupNCCL and other multi-stream code rely on it).  Called once
// after change_current_allocator installed this shim.
extern "C" int lms_torch_hook_record_stream() {
  auto a = torch::cuda::CUDAPluggableAllocator::getCurrentAllocator();
  auto p = std::dynamic_pointer_cast<torch::cuda::CUDAPluggableAllocator::CUDAPluggableAllocator>(a);
  if (!p) return -1;
  p->set_record_stream_fn([](void* ptr, cudaStream_t stream) {
    lms_ctx* c = lms_get_global();
    if (c) lms_dev_record_stream(c, ptr, stream);
  });
  return 0;
}
