// k_tile instantiations for group width ≤ 64 (FP32-strict and tcgen05 TF32).
#include "tile.cuh"

namespace gsrk {

cudaError_t launch_tile_w64(const TileArgs& a, cudaStream_t s, int* g) {
    return a.tc ? tile::launch_w<64, 1>(a, s, g) : tile::launch_w<64, 0>(a, s, g);
}

cudaError_t init_tile_w64() {
    const cudaError_t e0 = tile::set_attrs<64, 0>();
    const cudaError_t e1 = tile::set_attrs<64, 1>();
    return e0 != cudaSuccess ? e0 : e1;
}

}  // namespace gsrk
