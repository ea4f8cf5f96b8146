// ft_torch_alloc.cpp -- ft_options.alloc / .free hooks (include/ft.h) backed
// by PyTorch's CUDA caching allocator, so that every device buffer of a libft
// handle (cost tables, wave arenas, pipeline scratch) is torch memory: it
// shows in torch.cuda.memory_allocated() and is reused across graphs without
// driver calls.  Built as a separate library (libft_torch_alloc.so) so that
// libft itself has no torch dependency; the Python binding passes these two
// function pointers through ft_options.
#include <cstddef>

#include <c10/cuda/CUDACachingAllocator.h>

extern "C" {

// alloc(bytes, stream, ctx): a block of the current device, associated with
// `stream` (stream-ordered reuse inside the caching allocator); NULL on OOM.
void* ft_torch_alloc(size_t bytes, void* stream, void* /*ctx*/) {
  try {
    return c10::cuda::CUDACachingAllocator::raw_alloc_with_stream(bytes, (cudaStream_t)stream);
  } catch (...) {
    return nullptr;
  }
}

// free(p, stream, ctx): back to the cache; the block's stream is the one it
// was allocated on, which is the handle's only stream.
void ft_torch_free(void* p, void* /*stream*/, void* /*ctx*/) {
  try {
    c10::cuda::CUDACachingAllocator::raw_delete(p);
  } catch (...) {
  }
}

}  // extern "C"
