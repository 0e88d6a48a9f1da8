// C-ABI: the fused DMA forward (placeholder until the sm_100a kernel lands).
#include "common.cuh"

static thread_local int g_launches = 0;

extern "C" {
size_t dma_attention_workspace_bytes(const DmaAttnArgs*) { return 0; }
int dma_attention_supported(const DmaAttnArgs*) { return DMA_EUNSUPPORTED; }
int dma_attention_quantize(const DmaAttnArgs*, void*) { return DMA_EUNSUPPORTED; }
int dma_attention_core(const DmaAttnArgs*, void*) { return DMA_EUNSUPPORTED; }
int dma_attention_fwd(const DmaAttnArgs*, void*) { return DMA_EUNSUPPORTED; }
int dma_last_launch_count(void) { return g_launches; }
}
