// bulk_copy.cuh — PTX wrappers for the bulk-async copy engine (TMA, 1D form) and the shared-memory
// mbarriers its completion is counted on. SASS: UBLKCP for the copies, SYNCS for the barrier operations.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace slabgpu {
	namespace kern {
		namespace bulk {

			__device__ __forceinline__ uint32_t smem_u32( const void * p ) {
				return static_cast< uint32_t >( __cvta_generic_to_shared( p ) );
			}
			__device__ __forceinline__ void mbar_init( uint64_t * bar, unsigned int count ) {
				asm volatile( "mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"( smem_u32( bar ) ), "r"( count ) : "memory" );
			}
			__device__ __forceinline__ void mbar_fence_init() {
				asm volatile( "fence.mbarrier_init.release.cluster;" ::: "memory" );
			}
			__device__ __forceinline__ void mbar_arrive_expect_tx( uint64_t * bar, unsigned int bytes ) {
				asm volatile( "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"( smem_u32( bar ) ), "r"( bytes ) : "memory" );
			}
			__device__ __forceinline__ void mbar_arrive( uint64_t * bar ) {
				asm volatile( "mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"( smem_u32( bar ) ) : "memory" );
			}
			__device__ __forceinline__ void mbar_wait( uint64_t * bar, unsigned int parity ) {
				asm volatile(
					"{\n"
					".reg .pred P1;\n"
					"LAB_WAIT:\n"
					"mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
					"@P1 bra DONE;\n"
					"bra LAB_WAIT;\n"
					"DONE:\n"
					"}" ::"r"( smem_u32( bar ) ),
					"r"( parity )
					: "memory" );
			}
			// global -> shared bulk copy; `bytes` a multiple of 16, both addresses 16-byte aligned; completion is
			// counted in bytes on `bar`
			__device__ __forceinline__ void g2s( void * dst, const void * src, unsigned int bytes, uint64_t * bar ) {
				asm volatile( "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"( smem_u32( dst ) ),
					"l"( __cvta_generic_to_global( src ) ), "r"( bytes ), "r"( smem_u32( bar ) )
					: "memory" );
			}
			// shared -> global bulk copy, tracked by the issuing thread's bulk async-group
			__device__ __forceinline__ void s2g( void * dst, const void * src, unsigned int bytes ) {
				asm volatile( "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"( __cvta_generic_to_global( dst ) ), "r"( smem_u32( src ) ),
					"r"( bytes )
					: "memory" );
			}
			__device__ __forceinline__ void commit_group() {
				asm volatile( "cp.async.bulk.commit_group;" ::: "memory" );
			}
			// every committed group of this thread has finished READING its shared-memory source
			__device__ __forceinline__ void wait_group_read0() {
				asm volatile( "cp.async.bulk.wait_group.read 0;" ::: "memory" );
			}
			// every committed group of this thread is complete
			__device__ __forceinline__ void wait_group0() {
				asm volatile( "cp.async.bulk.wait_group 0;" ::: "memory" );
			}
			// generic-proxy accesses to shared memory before this point are ordered before later async-proxy ones
			__device__ __forceinline__ void fence_proxy_async() {
				asm volatile( "fence.proxy.async.shared::cta;" ::: "memory" );
			}

		} // namespace bulk
	} // namespace kern
} // namespace slabgpu
