// device_util.cuh — pieces shared by the kernel translation units: the programmatic-dependent-launch
// fences, the fixed-shape block reduction and the PDL launch helper.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "common.hpp"

namespace slabgpu {
	namespace kern {
		namespace dev {

			constexpr int kBlock = 256;

			inline unsigned int blocks_for( uint64_t count, int block = kBlock ) {
				return static_cast< unsigned int >( ( count + block - 1 ) / block );
			}

			// wait until the previous kernel in the stream has completed and its writes are visible
			__device__ __forceinline__ void dep_wait() {
				asm volatile( "griddepcontrol.wait;" ::: "memory" );
			}
			// let the next kernel's blocks be scheduled as soon as SM resources free up
			__device__ __forceinline__ void dep_trigger() {
				asm volatile( "griddepcontrol.launch_dependents;" ::: "memory" );
			}

			// fixed-shape tree reduction: shuffle tree per warp, shared-memory tree per block
			// (smem: 32 doubles). The result is valid in thread 0.
			__device__ __forceinline__ double block_tree_sum( double v, double * smem ) {
				#pragma unroll
				for( int off = 16; off > 0; off >>= 1 ) {
					v = __dadd_rn( v, __shfl_down_sync( 0xffffffffu, v, off ) );
				}
				const int warp = threadIdx.x >> 5;
				const int lane = threadIdx.x & 31;
				if( lane == 0 ) {
					smem[ warp ] = v;
				}
				__syncthreads();
				const int nwarps = blockDim.x >> 5;
				v = threadIdx.x < nwarps ? smem[ threadIdx.x ] : 0.0;
				if( warp == 0 ) {
					#pragma unroll
					for( int off = 16; off > 0; off >>= 1 ) {
						v = __dadd_rn( v, __shfl_down_sync( 0xffffffffu, v, off ) );
					}
				}
				__syncthreads();
				return v;
			}

			// launch with the programmatic-stream-serialization attribute (when enabled)
			template< class... KArgs, class... Args >
			void launch_pdl( void ( *kernel )( KArgs... ), unsigned int grid, unsigned int block, cudaStream_t st,
				Args... args ) {
				cudaLaunchConfig_t cfg{};
				cfg.gridDim = dim3( grid, 1, 1 );
				cfg.blockDim = dim3( block, 1, 1 );
				cfg.dynamicSmemBytes = 0;
				cfg.stream = st;
				cudaLaunchAttribute attr[ 1 ];
				unsigned int count = 0;
				if( g_use_pdl ) {
					attr[ count ].id = cudaLaunchAttributeProgrammaticStreamSerialization;
					attr[ count ].val.programmaticStreamSerializationAllowed = 1;
					++count;
				}
				cfg.attrs = attr;
				cfg.numAttrs = count;
				SLAB_CUDA( cudaLaunchKernelEx( &cfg, kernel, static_cast< KArgs >( args )... ) );
				count_launch();
			}

		} // namespace dev
	} // namespace kern
} // namespace slabgpu
