// kernels.cu — hand-written sm_100a kernels of the CG+MG hot path.
//
// Arithmetic contract: the reference is compiled without FMA
// (proj/CMakeLists.txt:8-14), so every product is rounded before it is added. All fp64
// arithmetic below goes through __dmul_rn/__dadd_rn/__ddiv_rn, which the compiler never
// contracts, and the file is additionally built with -fmad=false.
//
// Performance shape. Every kernel here is an HBM-bound (fine level) or latency-bound (coarse
// levels) streaming kernel; none has GEMM shape, so no tensor-core path exists.
//  * The matrix stream of a row (values + 32-bit columns, 12 B per stored entry) is immutable, so
//    a thread issues ALL of its matrix loads up front, with a streaming (evict-first) hint that keeps
//    the 126 MB L2 for the vectors. That gives each thread ~324 B in flight.
//  * Kernels are chained with programmatic dependent launch: a kernel's blocks become resident
//    and preload their matrix rows while the previous kernel drains; `griddepcontrol.wait` then
//    orders every access to mutable data (vectors, scalars) after the previous kernel's writes.
//    EVERY kernel executes the wait before touching mutable memory, so ordering is transitive.
//    Pointers to data an earlier kernel of the stream may have written (vectors, scalars, partials) are
//    never `const __restrict__`: such loads become read-only-path loads that the compiler may hoist above
//    the wait (it did, once, in the exact dot: right results without PDL, wrong ones with it). Only the
//    immutable matrix data (values, columns, codes, row lists, masks) is __restrict__.
//  * Vector gathers (x / z) are served by L1/L2.
#include "kernels.cuh"

#include <atomic>

#include <cuda_runtime.h>

#include "common.hpp"
#include "bulk_copy.cuh"
#include "device_util.cuh"

namespace slabgpu {

	std::atomic< uint64_t > g_launch_count{ 0 };
	int g_use_pdl = 1;
	// L2 persisting carve-out (set by slab_ctx_create from the device limits; 0 = unused)
	size_t g_l2_persist_bytes = 0;
	int g_dot_cpb = 0; // exact dot: chunks per block (0 = spread the chunks over the SMs once)
	int g_dot_tile = 0; // exact dot: products per chunk and stage (0 = automatic)
	size_t g_l2_window_max = 0;
	// attach an access-policy window on z to fine-level colour steps. OFF by default: measured on B200
	// (tools/l2_window_probe.py) the carve-out helps the 192^3 sweep by 2.6% but costs 12-18% at 104^3 and
	// 256^3, because it shrinks the L2 that everything else shares. Enable with SLAB_L2_WINDOW=1.
	int g_l2_window = 0;
	uint64_t g_tuning_epoch = 0;
	// launches with at least this many rows use the streaming kernels, smaller ones the preload
	// kernels (measured cross-over on B200: between 1.4e5 and 8.8e5 rows per launch)
	int64_t g_stream_rows = 200000;
	// which streaming kernel shape the many-wave launches use (tuning knob). 2 = batches of 9 slots,
	// 48 registers, 40 resident warps per SM: best of the sweep in profiles/r01_microbench_*.json
	int g_stream_variant = 2;

	namespace kern {

		namespace {

			using namespace dev; // kBlock, blocks_for, dep_wait, dep_trigger, block_tree_sum
			constexpr int kChunk = 27; // slots preloaded per row in one go (a full 27-point row)

			// Vector that the next launch should keep in the L2 persisting carve-out (the z of a fine-level
			// colour step: every step gathers all of it while the matrix streams through). Consumed by the
			// next launch() only.
			thread_local const void * t_window_base = nullptr;
			size_t t_window_bytes = 0;

			// launch with the programmatic-stream-serialization attribute (PDL)
			template< class... KArgs, class... Args >
			void launch( void ( *kernel )( KArgs... ), unsigned int grid, unsigned int block, cudaStream_t st,
				Args... args ) {
				cudaLaunchConfig_t cfg{};
				cfg.gridDim = dim3( grid, 1, 1 );
				cfg.blockDim = dim3( block, 1, 1 );
				cfg.dynamicSmemBytes = 0;
				cfg.stream = st;
				cudaLaunchAttribute attr[ 2 ];
				unsigned int count = 0;
				if( g_use_pdl ) {
					attr[ count ].id = cudaLaunchAttributeProgrammaticStreamSerialization;
					attr[ count ].val.programmaticStreamSerializationAllowed = 1;
					++count;
				}
				if( t_window_base != nullptr && g_l2_persist_bytes > 0 ) {
					const size_t bytes = t_window_bytes < g_l2_window_max ? t_window_bytes : g_l2_window_max;
					attr[ count ].id = cudaLaunchAttributeAccessPolicyWindow;
					attr[ count ].val.accessPolicyWindow.base_ptr = const_cast< void * >( t_window_base );
					attr[ count ].val.accessPolicyWindow.num_bytes = bytes;
					const double ratio = static_cast< double >( g_l2_persist_bytes ) / static_cast< double >( bytes );
					attr[ count ].val.accessPolicyWindow.hitRatio = static_cast< float >( ratio < 1.0 ? ratio : 1.0 );
					attr[ count ].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
					attr[ count ].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
					++count;
				}
				t_window_base = nullptr;
				cfg.attrs = attr;
				cfg.numAttrs = count;
				SLAB_CUDA( cudaLaunchKernelEx( &cfg, kernel, static_cast< KArgs >( args )... ) );
				count_launch();
			}

			// ------------------------------------------------------------ SELL row access

			struct RowChunk {
				double v[ kChunk ];
				int32_t c[ kChunk ];
			};

			// entries [first, first+count) of the row at position `pos`: issue all loads, no use yet
			__device__ __forceinline__ void chunk_load( const double * __restrict__ vals, const int32_t * __restrict__ cols,
				int64_t at, int count, RowChunk & rc ) {
				#pragma unroll
				for( int k = 0; k < kChunk; ++k ) { // predicated loads, no branches: slots beyond the slice read as padding
					const bool in = k < count;
					rc.c[ k ] = in ? __ldcs( cols + at + static_cast< int64_t >( k ) * kSlice ) : -1;
					rc.v[ k ] = in ? __ldcs( vals + at + static_cast< int64_t >( k ) * kSlice ) : 0.0;
				}
			}

			// ordered accumulation acc = acc + v*x[c] over the chunk's stored entries, ascending
			// column order (operations.hpp:116-125); padding slots (c < 0) are skipped. All gathers
			// are issued before the dependent add chain starts.
			template< bool WANT_DIAG >
			__device__ __forceinline__ double chunk_accumulate( const RowChunk & rc, int count, const double * x, double acc,
				int32_t diag_row, double & diag ) {
				constexpr int kBatch = 9; // gathers in flight per thread while the add chain runs
				#pragma unroll
				for( int k0 = 0; k0 < kChunk; k0 += kBatch ) {
					double xv[ kBatch ];
					// straight-line code: slots beyond `count` carry column -1 (chunk_load) and drop out
					// through the same select as stored padding
					#pragma unroll
					for( int j = 0; j < kBatch; ++j ) {
						const int k = k0 + j;
						xv[ j ] = x[ rc.c[ k ] < 0 ? 0 : rc.c[ k ] ];
					}
					#pragma unroll
					for( int j = 0; j < kBatch; ++j ) {
						const int k = k0 + j;
						const double sum = __dadd_rn( acc, __dmul_rn( rc.v[ k ], xv[ j ] ) );
						acc = rc.c[ k ] < 0 ? acc : sum;
						if( WANT_DIAG ) {
							diag = rc.c[ k ] == diag_row ? rc.v[ k ] : diag;
						}
					}
				}
				return acc;
			}

			// rows wider than one chunk (general matrices): remaining chunks, loaded after the wait
			template< bool WANT_DIAG >
			__device__ __forceinline__ double row_tail( const double * __restrict__ vals, const int32_t * __restrict__ cols,
				int64_t begin, int width, const double * x, double acc, int32_t diag_row, double & diag ) {
				for( int k0 = kChunk; k0 < width; k0 += kChunk ) {
					RowChunk rc;
					const int count = width - k0 < kChunk ? width - k0 : kChunk;
					chunk_load( vals, cols, begin + static_cast< int64_t >( k0 ) * kSlice, count, rc );
					acc = chunk_accumulate< WANT_DIAG >( rc, count, x, acc, diag_row, diag );
				}
				return acc;
			}

			// ------------------------------------------------------------ vector ops

			// 16-byte stores in a grid-stride loop: one 8-byte store per thread reaches only 1.9 TB/s on B200
			// (tools/vector_ops_probe.py). `head` leading elements (0 or 1) bring the rest to a 16-byte boundary.
			__global__ void __launch_bounds__( kBlock ) k_fill( double * v, uint64_t n, double value, uint64_t head ) {
				dep_trigger();
				dep_wait();
				const uint64_t tid = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				if( tid < head ) {
					v[ tid ] = value;
				}
				double2 * v2 = reinterpret_cast< double2 * >( v + head );
				const uint64_t pairs = ( n - head ) >> 1;
				const double2 both = make_double2( value, value );
				for( uint64_t i = tid; i < pairs; i += stride ) {
					v2[ i ] = both;
				}
				if( tid == 0 && ( ( n - head ) & 1 ) ) {
					v[ n - 1 ] = value;
				}
			}

			// operations.hpp:103 — w may alias x or y: each thread reads its inputs before writing.
			// Two elements per thread and iteration through 16-byte accesses (all vectors start on 256-byte
			// boundaries); the arithmetic per element is unchanged.
			__global__ void __launch_bounds__( kBlock ) k_waxpby( double * w, double alpha, const double * x, double beta,
				const double * y, uint64_t n ) {
				dep_trigger();
				dep_wait();
				const uint64_t tid = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				const uint64_t pairs = n >> 1;
				for( uint64_t i = tid; i < pairs; i += stride ) {
					const double2 xv = reinterpret_cast< const double2 * >( x )[ i ];
					const double2 yv = reinterpret_cast< const double2 * >( y )[ i ];
					double2 out;
					out.x = __dadd_rn( __dmul_rn( alpha, xv.x ), __dmul_rn( beta, yv.x ) );
					out.y = __dadd_rn( __dmul_rn( alpha, xv.y ), __dmul_rn( beta, yv.y ) );
					reinterpret_cast< double2 * >( w )[ i ] = out;
				}
				if( tid == 0 && ( n & 1 ) ) {
					w[ n - 1 ] = __dadd_rn( __dmul_rn( alpha, x[ n - 1 ] ), __dmul_rn( beta, y[ n - 1 ] ) );
				}
			}

			// operations.hpp:61-91: one warp per 4096-element chunk. The chunk's rounded products are added left
			// to right by lane 0 — a chain of 4096 dependent additions (8.8 cycles each on B200,
			// tools/probes/fp64_latency.cu), which is what this kernel costs. Everything else hides behind it:
			// the chunk moves through shared memory in tiles of 512 products, and while lane 0 adds one tile all
			// 32 lanes already hold the loads of the next tile in flight. 8 KB of shared memory per warp keeps
			// every chunk of a 192^3 vector resident at once. The block that finishes last adds the per-chunk
			// partials in chunk order.
			constexpr int kDotTile = 512;
			// acc + p[0] + p[1] + ... left to right, for ONE thread. The additions form a dependent chain; the
			// shared-memory reads must not sit in it, so the next 16 values are in registers before the
			// current 16 are added (the compiler does not pipeline this by itself: 19 cycles per element
			// instead of the 8.8 of the addition alone).
			__device__ __forceinline__ double chain_sum( const double * p, int count, double acc ) {
				constexpr int kStep = 16;
				double ra[ kStep ], rb[ kStep ]; // two register sets that swap roles statically (no copies)
				#pragma unroll
				for( int k = 0; k < kStep; ++k ) {
					ra[ k ] = k < count ? p[ k ] : 0.0;
				}
				int i = 0;
				for( ; i + 2 * kStep <= count; i += 2 * kStep ) {
					#pragma unroll
					for( int k = 0; k < kStep; ++k ) {
						rb[ k ] = p[ i + kStep + k ];
					}
					#pragma unroll
					for( int k = 0; k < kStep; ++k ) {
						acc = __dadd_rn( acc, ra[ k ] );
					}
					#pragma unroll
					for( int k = 0; k < kStep; ++k ) {
						ra[ k ] = i + 2 * kStep + k < count ? p[ i + 2 * kStep + k ] : 0.0;
					}
					#pragma unroll
					for( int k = 0; k < kStep; ++k ) {
						acc = __dadd_rn( acc, rb[ k ] );
					}
				}
				// fewer than 32 left: ra holds the next 16 (zero beyond count)
				#pragma unroll
				for( int k = 0; k < kStep; ++k ) {
					if( i + k < count ) {
						acc = __dadd_rn( acc, ra[ k ] );
					}
				}
				for( int j = i + kStep; j < count; ++j ) {
					acc = __dadd_rn( acc, p[ j ] );
				}
				return acc;
			}

			// One LANE per chunk. A chain of 4096 dependent additions costs 4096 x 8.8 cycles whoever runs it, and a warp
			// instruction with one active lane takes the FP64 pipe's issue slot like a full one — so the chunks an SM is
			// responsible for ride in the lanes of ONE warp (lane c adds chunk c: up to 32 chains per instruction), and
			// that warp does nothing but read a product and add it: every other instruction in it costs chain time (the
			// multiply next to the add nearly doubled it). The block's other three warps sit on the other three
			// sub-partitions and feed it: the operands arrive by the bulk-async copy engine (each chunk's next tiles of x
			// and y, two contiguous pieces per tile, into a three-stage ring, completion counted on the stage's
			// mbarrier), the converter warps round the products on their own (operations.hpp:74) into a two-deep ring of
			// product tiles, and full/empty mbarriers hand the tiles over. Rows of the rings are tile + 2 (raw: 16-byte
			// aligned for the copies) and tile + 1 (products: the lanes' reads fall into different banks) doubles apart.
			// The block that finishes last adds the per-chunk partials in chunk order (operations.hpp:84-90).
			constexpr int kDotStages = 3;
			constexpr int kDotThreads = 128; // warp 0 adds; warps 1..3 copy and multiply

			__global__ void __launch_bounds__( kDotThreads ) k_dot_exact( const double * x, const double * y, uint64_t n, int cpb, int tile, double * partials,
				unsigned int * counter, double * out ) {
				extern __shared__ __align__( 128 ) unsigned char dot_smem[];
				uint64_t * const full_raw = reinterpret_cast< uint64_t * >( dot_smem );     // [kDotStages]
				uint64_t * const full_prod = full_raw + kDotStages;                          // [2]
				uint64_t * const empty_prod = full_prod + 2;                                 // [2]
				__shared__ bool is_last;
				const int t = threadIdx.x;
				const int lane = t & 31;
				const int pitch = tile + 2, ppitch = tile + 1;
				const size_t stage_elems = static_cast< size_t >( 2 ) * cpb * pitch;
				double * const raw0 = reinterpret_cast< double * >( dot_smem + 128 );       // [kDotStages][2][cpb][pitch]
				double * const prod0 = raw0 + kDotStages * stage_elems;                      // [2][cpb][ppitch]
				if( t == 0 ) {
					for( int s = 0; s < kDotStages; ++s ) {
						bulk::mbar_init( full_raw + s, 1u );
					}
					for( int s = 0; s < 2; ++s ) {
						bulk::mbar_init( full_prod + s, 3u );  // one arrival per converter warp
						bulk::mbar_init( empty_prod + s, 1u ); // the adding warp
					}
					bulk::mbar_fence_init();
				}
				__syncthreads();
				dep_trigger();
				dep_wait();
				const uint64_t nchunks = ( n + kDotChunk - 1 ) / kDotChunk;
				const uint64_t chunk0 = static_cast< uint64_t >( blockIdx.x ) * cpb;
				const int nmine = static_cast< int >( nchunks - chunk0 < static_cast< uint64_t >( cpb ) ? nchunks - chunk0 : cpb );
				// tiles of the block's longest chunk (its first: only the last chunk of the vector is short)
				const uint64_t longest = n - chunk0 * kDotChunk < kDotChunk ? n - chunk0 * kDotChunk : kDotChunk;
				const int ntiles = static_cast< int >( ( longest + tile - 1 ) / tile );

				if( t < 32 ) {
					// ------------------------------------------------ the adding warp: lane c walks chunk c's products
					double acc = 0.0;
					#pragma unroll 1
					for( int k = 0; k < ntiles; ++k ) {
						const int b = k & 1;
						bulk::mbar_wait( full_prod + b, static_cast< unsigned int >( ( k >> 1 ) & 1 ) );
						if( lane < nmine ) {
							acc = chain_sum( prod0 + ( static_cast< size_t >( b ) * cpb + lane ) * ppitch, tile, acc );
						}
						__syncwarp();
						if( lane == 0 ) {
							bulk::mbar_arrive( empty_prod + b );
						}
					}
					if( lane < nmine ) {
						partials[ chunk0 + lane ] = acc;
					}
					__threadfence();
				} else {
					// ------------------------------------------------ the converter warps
					const int ct = t - 32; // 0..95
					const bool issuer = t < 64; // lanes of warp 1 own the copy engine: lane c <-> chunk c
					const uint64_t begin = ( chunk0 + lane ) * kDotChunk;
					const int len = ( issuer && lane < nmine ) ? static_cast< int >( n - begin < kDotChunk ? n - begin : kDotChunk ) : 0;
					const bool aligned = ( ( reinterpret_cast< uintptr_t >( x ) | reinterpret_cast< uintptr_t >( y ) ) & 15 ) == 0;
					// tile k of every chunk of the block into raw stage k % kDotStages: whole, 16-byte-aligned pieces by bulk
					// copies, a ragged or unaligned piece by the lane itself (+0.0 behind the end of the vector: adding a +0.0
					// product to a sum that started from +0.0 changes nothing)
					const auto issue = [ & ]( int k ) {
						const int s = k % kDotStages;
						double * const xs = raw0 + s * stage_elems + static_cast< size_t >( lane ) * pitch;
						double * const ys = xs + static_cast< size_t >( cpb ) * pitch;
						const int have = len - k * tile < 0 ? 0 : ( len - k * tile < tile ? len - k * tile : tile );
						const bool by_copy = aligned && have == tile;
						unsigned int bytes = by_copy ? static_cast< unsigned int >( tile ) * 16u : 0u;
						#pragma unroll
						for( int o = 16; o > 0; o >>= 1 ) {
							bytes += __shfl_xor_sync( 0xffffffffu, bytes, o );
						}
						if( lane < nmine && !by_copy ) {
							for( int i = 0; i < tile; ++i ) {
								xs[ i ] = i < have ? x[ begin + static_cast< uint64_t >( k ) * tile + i ] : 0.0;
								ys[ i ] = i < have ? y[ begin + static_cast< uint64_t >( k ) * tile + i ] : 0.0;
							}
						}
						__syncwarp();
						if( lane == 0 ) {
							if( bytes > 0u ) {
								bulk::mbar_arrive_expect_tx( full_raw + s, bytes );
							} else {
								bulk::mbar_arrive( full_raw + s );
							}
						}
						__syncwarp();
						if( by_copy ) {
							bulk::g2s( xs, x + begin + static_cast< uint64_t >( k ) * tile, static_cast< unsigned int >( tile ) * 8u, full_raw + s );
							bulk::g2s( ys, y + begin + static_cast< uint64_t >( k ) * tile, static_cast< unsigned int >( tile ) * 8u, full_raw + s );
						}
					};
					if( issuer ) {
						for( int k = 0; k < kDotStages && k < ntiles; ++k ) {
							issue( k );
						}
					}
					#pragma unroll 1
					for( int k = 0; k < ntiles; ++k ) {
						const int s = k % kDotStages, b = k & 1;
						bulk::mbar_wait( full_raw + s, static_cast< unsigned int >( ( k / kDotStages ) & 1 ) );
						if( k >= 2 ) { // the adding warp is done with the product tile this one replaces
							bulk::mbar_wait( empty_prod + b, static_cast< unsigned int >( ( ( k >> 1 ) - 1 ) & 1 ) );
						}
						const double * const xs = raw0 + s * stage_elems;
						const double * const ys = xs + static_cast< size_t >( cpb ) * pitch;
						double * const pd = prod0 + static_cast< size_t >( b ) * cpb * ppitch;
						const int total = nmine * tile;
						for( int idx = ct; idx < total; idx += kDotThreads - 32 ) {
							const int c = idx / tile, i = idx - c * tile;
							pd[ c * ppitch + i ] = __dmul_rn( xs[ c * pitch + i ], ys[ c * pitch + i ] );
						}
						__syncwarp();
						if( lane == 0 ) {
							bulk::mbar_arrive( full_prod + b );
						}
						// the raw stage is free once all three converter warps have read it
						asm volatile( "bar.sync 2, 96;" ::: "memory" );
						if( issuer && k + kDotStages < ntiles ) {
							bulk::fence_proxy_async();
							issue( k + kDotStages );
						}
					}
				}
				__syncthreads();
				if( t == 0 ) {
					is_last = atomicAdd( counter, 1u ) == gridDim.x - 1;
				}
				__syncthreads();
				if( !is_last ) {
					return;
				}
				// the block that finishes last adds the per-chunk partials in chunk order: a chain for thread 0, fed through
				// shared memory in tiles that all threads fetch together
				__threadfence();
				const size_t have_doubles = kDotStages * stage_elems + static_cast< size_t >( 2 ) * cpb * ppitch;
				const int room = static_cast< int >( have_doubles < 4096 ? have_doubles : 4096 );
				double total = 0.0;
				for( uint64_t t0 = 0; t0 < nchunks; t0 += room ) {
					const int m = static_cast< int >( nchunks - t0 < static_cast< uint64_t >( room ) ? nchunks - t0 : room );
					__syncthreads();
					for( int i = t; i < m; i += kDotThreads ) {
						raw0[ i ] = __ldcg( partials + t0 + i );
					}
					__syncthreads();
					if( t == 0 ) {
						total = chain_sum( raw0, m, total );
					}
				}
				if( t == 0 ) {
					*out = total;
					*counter = 0u;
				}
			}

			__global__ void k_dot_empty( double * out ) {
				dep_trigger();
				dep_wait();
				*out = 0.0;
			}

			// fixed-shape tree reduction: grid-stride partial per thread, block_tree_sum per block,
			// last block folds the block partials the same way.
			__device__ __forceinline__ void grid_tree_finish( double block_sum, double * partials, unsigned int * counter,
				double * out, double * smem, bool * is_last ) {
				if( threadIdx.x == 0 ) {
					partials[ blockIdx.x ] = block_sum;
					__threadfence();
					const unsigned int ticket = atomicAdd( counter, 1u );
					*is_last = ticket == gridDim.x - 1;
				}
				__syncthreads();
				if( *is_last ) {
					__threadfence();
					double v = 0.0;
					for( unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x ) {
						v = __dadd_rn( v, __ldcg( partials + b ) );
					}
					v = block_tree_sum( v, smem );
					if( threadIdx.x == 0 ) {
						*out = v;
						*counter = 0u;
					}
				}
			}

			// one block folds `count` block partials in a fixed order (each thread a strided chain, then the tree)
			__global__ void __launch_bounds__( 1024 ) k_sum_partials( const double * partials, uint64_t count,
				double * out ) {
				__shared__ double smem[ 32 ];
				dep_trigger();
				dep_wait();
				double v = 0.0;
				for( uint64_t b = threadIdx.x; b < count; b += blockDim.x ) {
					v = __dadd_rn( v, partials[ b ] );
				}
				v = block_tree_sum( v, smem );
				if( threadIdx.x == 0 ) {
					*out = v;
				}
			}

			__global__ void __launch_bounds__( kBlock ) k_dot_tree( const double * x,
				const double * y, uint64_t n, double * partials, unsigned int * counter, double * out ) {
				__shared__ double smem[ 32 ];
				__shared__ bool is_last;
				dep_trigger();
				dep_wait();
				// 16-byte loads, two pairs in flight per thread and iteration; four independent chains
				double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				const uint64_t pairs = n >> 1;
				const double2 * x2 = reinterpret_cast< const double2 * >( x );
				const double2 * y2 = reinterpret_cast< const double2 * >( y );
				uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				for( ; i + stride < pairs; i += 2 * stride ) {
					const double2 a0 = x2[ i ], b0 = y2[ i ];
					const double2 a1 = x2[ i + stride ], b1 = y2[ i + stride ];
					acc0 = __dadd_rn( acc0, __dmul_rn( a0.x, b0.x ) );
					acc1 = __dadd_rn( acc1, __dmul_rn( a0.y, b0.y ) );
					acc2 = __dadd_rn( acc2, __dmul_rn( a1.x, b1.x ) );
					acc3 = __dadd_rn( acc3, __dmul_rn( a1.y, b1.y ) );
				}
				for( ; i < pairs; i += stride ) {
					const double2 a0 = x2[ i ], b0 = y2[ i ];
					acc0 = __dadd_rn( acc0, __dmul_rn( a0.x, b0.x ) );
					acc1 = __dadd_rn( acc1, __dmul_rn( a0.y, b0.y ) );
				}
				if( blockIdx.x == 0 && threadIdx.x == 0 && ( n & 1 ) ) {
					acc2 = __dadd_rn( acc2, __dmul_rn( x[ n - 1 ], y[ n - 1 ] ) );
				}
				const double acc = __dadd_rn( __dadd_rn( acc0, acc1 ), __dadd_rn( acc2, acc3 ) );
				grid_tree_finish( block_tree_sum( acc, smem ), partials, counter, out, smem, &is_last );
			}

			// ------------------------------------------------------------ SELL products

			// operations.hpp:164-174. MASKED: one thread per mask member, others untouched.
			template< bool MASKED >
			__global__ void __launch_bounds__( kBlock ) k_spmv( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const double * x,
				double * y, const int32_t * __restrict__ members, int64_t count, double * dot_partials,
				unsigned int * dot_counter, double * dot_out ) {
				__shared__ double smem[ 32 ];
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const bool live = k < count;
				int64_t row = 0, begin = 0;
				int width = 0;
				RowChunk rc;
				if( live ) {
					row = MASKED ? members[ k ] : k;
					const int64_t s = row >> 5;
					const int64_t b = slice_off[ s ];
					width = static_cast< int >( ( slice_off[ s + 1 ] - b ) >> 5 );
					begin = b + ( row & 31 );
					chunk_load( vals, cols, begin, width < kChunk ? width : kChunk, rc );
				}
				dep_trigger();
				dep_wait();
				double prod = 0.0;
				if( live ) {
					double unused = 0.0;
					double acc = chunk_accumulate< false >( rc, width < kChunk ? width : kChunk, x, 0.0, -1, unused );
					acc = row_tail< false >( vals, cols, begin, width, x, acc, -1, unused );
					y[ row ] = acc;
					prod = dot_out != nullptr ? __dmul_rn( x[ row ], acc ) : 0.0;
				}
				if( dot_out != nullptr ) { // x'(A x): block partials here, folded by k_sum_partials (cg.hpp:122-123)
					const double block_sum = block_tree_sum( prod, smem );
					if( threadIdx.x == 0 ) {
						dot_partials[ blockIdx.x ] = block_sum;
					}
				}
			}

			// smoother.hpp:60-72 fused: s = row sum over z, then z[i] = ((r[i] - s) + z[i]*d) / d.
			// Rows of one colour never neighbour each other, so reading z while other threads of
			// the same launch write their own z[i] is race-free (coloring.hpp:165-204).
			// Grid transfers ride on the colour-0 steps next to them (stencil levels: colour 0 == injected rows,
			// position k of the colour-0 block == coarse row k):
			//  flags & 1 — prolongation first (multigrid.hpp:71-81): z[i] <- 1*z[i] + 1*(0 + 1*src[k]); the
			//    value is stored before the row sum, whose diagonal gather then reads it back;
			//  flags & 2 — residual + restriction behind (multigrid.hpp:100-104), valid on the LAST backward
			//    colour-0 step where every other colour is final: with the new z[i] stored, the ordered row sum
			//    is taken again (matrix row still in registers) and out[k] = 0 + 1*(1*r[i] + (-1)*(A z)[i]);
			//    zero[k] = 0 prepares the coarse guess (multigrid.hpp:104).
			__global__ void __launch_bounds__( kBlock, 2 ) k_gs_color( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t pos_begin, int64_t pos_count, double * z, const double * r, int flags,
				const double * src, double * out, double * zero,
				const int32_t * __restrict__ pos_list, const uint8_t * __restrict__ skip ) {
				// pos_list: the launch covers exactly these positions (the boundary rows of a colour, computed
				// first so that their halo messages travel while the interior rows run); skip: positions
				// flagged here are left out (the interior launch of the same colour)
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				int32_t i = -1;
				int64_t begin = 0;
				int64_t coarse = 0;
				int width = 0;
				RowChunk rc;
				if( k < pos_count ) {
					const int64_t pos = pos_list != nullptr ? pos_list[ k ] : pos_begin + k;
					coarse = pos - pos_begin;
					i = skip != nullptr && skip[ pos ] ? -1 : rows[ pos ];
					const int64_t s = pos >> 5;
					const int64_t b = slice_off[ s ];
					width = static_cast< int >( ( slice_off[ s + 1 ] - b ) >> 5 );
					begin = b + ( pos & 31 );
					chunk_load( vals, cols, begin, width < kChunk ? width : kChunk, rc );
				}
				dep_trigger();
				dep_wait();
				if( i < 0 ) {
					return;
				}
				const double ri = r[ i ];
				double zi = z[ i ];
				if( flags & 1 ) {
					const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ coarse ] ) );
					zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
					z[ i ] = zi;
				}
				// flags & 4 — the step runs twice in a row (the last colour of the forward sweep is the first of the
				//    backward sweep, smoother.hpp:108-111): nothing but z[i] itself changes in between, so the same
				//    thread repeats the ordered row sum and the update with the matrix row still in registers.
				const int passes = ( flags & 4 ) ? 2 : 1;
				#pragma unroll 1
				for( int pass = 0; pass < passes; ++pass ) {
					double d = 0.0;
					double s = chunk_accumulate< true >( rc, width < kChunk ? width : kChunk, z, 0.0, i, d );
					s = row_tail< true >( vals, cols, begin, width, z, s, i, d );
					zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -s ), __dmul_rn( zi, d ) ), d );
					z[ i ] = zi;
				}
				if( flags & 2 ) {
					double unused = 0.0;
					double az = chunk_accumulate< false >( rc, width < kChunk ? width : kChunk, z, 0.0, -1, unused );
					az = row_tail< false >( vals, cols, begin, width, z, az, -1, unused );
					const double f = __dadd_rn( __dmul_rn( 1.0, ri ), __dmul_rn( -1.0, az ) );
					out[ coarse ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
					zero[ coarse ] = 0.0;
				}
			}

			// multigrid.hpp:100-104 fused on the injected rows (= the colour-0 block, whose p-th
			// member is the fine point of coarse index p): f = 1*r + (-1)*(A z), r_c = 0 + 1*f.
			__global__ void __launch_bounds__( kBlock ) k_residual_restrict( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t n_coarse, const double * z, const double * r,
				double * r_c, double * zero ) {
				const int64_t p = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const bool live = p < n_coarse;
				int32_t i = 0;
				int64_t begin = 0;
				int width = 0;
				RowChunk rc;
				if( live ) {
					i = rows[ p ];
					const int64_t s = p >> 5;
					const int64_t b = slice_off[ s ];
					width = static_cast< int >( ( slice_off[ s + 1 ] - b ) >> 5 );
					begin = b + ( p & 31 );
					chunk_load( vals, cols, begin, width < kChunk ? width : kChunk, rc );
				}
				dep_trigger();
				dep_wait();
				if( !live ) {
					return;
				}
				double unused = 0.0;
				double az = chunk_accumulate< false >( rc, width < kChunk ? width : kChunk, z, 0.0, -1, unused );
				az = row_tail< false >( vals, cols, begin, width, z, az, -1, unused );
				const double f = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -1.0, az ) );
				r_c[ p ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
				if( zero != nullptr ) {
					zero[ p ] = 0.0; // set_all(z_c, 0), multigrid.hpp:104
				}
			}

			// Batched streaming row sum: B (column, value) pairs are loaded together, then their B
			// gathers, then the B-long ordered add chain; the next batch's matrix loads are issued
			// before the chain of the current one runs (software pipelining by hand).
			// COHERENT: gather x through L2 only (ld.global.cg) — needed inside the persistent V-cycle
			// kernel, where other SMs update x between grid barriers and L1 would serve stale lines.
			template< int B, bool WANT_DIAG, bool COHERENT = false >
			__device__ __forceinline__ double row_sum_batched( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, int64_t pos, const double * x,
				int32_t diag_row, double & diag ) {
				const int64_t s = pos >> 5;
				const int64_t base = slice_off[ s ];
				const int width = static_cast< int >( ( slice_off[ s + 1 ] - base ) >> 5 );
				const double * vp = vals + base + ( pos & 31 );
				const int32_t * cp = cols + base + ( pos & 31 );
				double acc = 0.0;
				int32_t c[ B ];
				double v[ B ];
				#pragma unroll
				for( int j = 0; j < B; ++j ) {
					const bool in = j < width;
					c[ j ] = in ? __ldcs( cp + j * kSlice ) : -1;
					v[ j ] = in ? __ldcs( vp + j * kSlice ) : 0.0;
				}
				for( int k0 = 0; k0 < width; k0 += B ) {
					double xv[ B ];
					#pragma unroll
					for( int j = 0; j < B; ++j ) {
						const double * xp = x + ( c[ j ] < 0 ? 0 : c[ j ] );
						xv[ j ] = COHERENT ? __ldcg( xp ) : *xp;
					}
					int32_t cc[ B ];
					double vv[ B ];
					#pragma unroll
					for( int j = 0; j < B; ++j ) {
						cc[ j ] = c[ j ];
						vv[ j ] = v[ j ];
					}
					// next batch of matrix entries goes out before the dependent chain below
					#pragma unroll
					for( int j = 0; j < B; ++j ) {
						const int k = k0 + B + j;
						const bool in = k < width;
						c[ j ] = in ? __ldcs( cp + k * kSlice ) : -1;
						v[ j ] = in ? __ldcs( vp + k * kSlice ) : 0.0;
					}
					#pragma unroll
					for( int j = 0; j < B; ++j ) {
						const double sum = __dadd_rn( acc, __dmul_rn( vv[ j ], xv[ j ] ) );
						acc = cc[ j ] < 0 ? acc : sum;
						if( WANT_DIAG ) {
							diag = cc[ j ] == diag_row ? vv[ j ] : diag;
						}
					}
				}
				return acc;
			}

			template< int B, int MINBLOCKS >
			__global__ void __launch_bounds__( kBlock, MINBLOCKS ) k_gs_color_batched( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t pos_begin, int64_t pos_count, double * z, const double * r,
				const double * src, const int32_t * __restrict__ pos_list, const uint8_t * __restrict__ skip ) {
				dep_trigger();
				dep_wait();
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( k >= pos_count ) {
					return;
				}
				const int64_t pos = pos_list != nullptr ? pos_list[ k ] : pos_begin + k; // see k_gs_color
				if( skip != nullptr && skip[ pos ] ) {
					return;
				}
				const int32_t i = rows[ pos ];
				if( i < 0 ) {
					return;
				}
				double zi = z[ i ];
				if( src != nullptr ) { // prolongation fused in front, see k_gs_color
					const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ pos - pos_begin ] ) );
					zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
					z[ i ] = zi;
				}
				double d = 0.0;
				const double s = row_sum_batched< B, true >( slice_off, vals, cols, pos, z, i, d );
				const double ri = r[ i ];
				z[ i ] = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -s ), __dmul_rn( zi, d ) ), d );
			}

			template< int B, int MINBLOCKS >
			__global__ void __launch_bounds__( kBlock, MINBLOCKS ) k_spmv_batched( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const double * x,
				double * y, int64_t nrows, double * dot_partials, unsigned int * dot_counter, double * dot_out ) {
				__shared__ double smem[ 32 ];
				dep_trigger();
				dep_wait();
				const int64_t row = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				double prod = 0.0;
				if( row < nrows ) {
					double unused = 0.0;
					const double acc = row_sum_batched< B, false >( slice_off, vals, cols, row, x, -1, unused );
					y[ row ] = acc;
					prod = dot_out != nullptr ? __dmul_rn( x[ row ], acc ) : 0.0;
				}
				if( dot_out != nullptr ) { // x'(A x): block partials here, folded by k_sum_partials (cg.hpp:122-123)
					const double block_sum = block_tree_sum( prod, smem );
					if( threadIdx.x == 0 ) {
						dot_partials[ blockIdx.x ] = block_sum;
					}
				}
			}

			// ---- streaming forms (many-wave launches on the fine level); same arithmetic, same order

			__global__ void __launch_bounds__( kBlock ) k_residual_restrict_stream( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t n_coarse, const double * z, const double * r,
				double * r_c, double * zero ) {
				dep_trigger();
				dep_wait();
				const int64_t p = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( p >= n_coarse ) {
					return;
				}
				const int32_t i = rows[ p ];
				double unused = 0.0;
				const double az = row_sum_batched< 9, false >( slice_off, vals, cols, p, z, -1, unused );
				const double f = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -1.0, az ) );
				r_c[ p ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
				if( zero != nullptr ) {
					zero[ p ] = 0.0;
				}
			}

			// multigrid.hpp:71-81 at the injected rows: f[i] = 0 + 1*z_c[p]; z[i] = 1*z[i] + 1*f[i].
			// (Elsewhere the reference computes z + 0.0, which only turns -0.0 into +0.0.)
			__global__ void k_prolong_add( const int32_t * __restrict__ rows, int64_t n_coarse, double * z,
				const double * z_c ) {
				const int64_t p = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const int32_t i = p < n_coarse ? rows[ p ] : -1;
				dep_trigger();
				dep_wait();
				if( i < 0 ) {
					return;
				}
				const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, z_c[ p ] ) );
				z[ i ] = __dadd_rn( __dmul_rn( 1.0, z[ i ] ), __dmul_rn( 1.0, f ) );
			}

			// ------------------------------------------------------------ CG updates

			// hist_rr != nullptr (cg.cu, inline bookkeeping): thread 0 also writes the PREVIOUS iteration's history entry —
			// r'r and p'Ap still hold its values here — and the r update of this iteration bumps the counter, so no
			// launch is spent on bookkeeping
			__global__ void __launch_bounds__( kBlock ) k_cg_update_p( double * p, const double * z,
				const double * scalars, const unsigned int * iter_counter, uint64_t n, double * hist_rr, double * hist_pq ) {
				dep_trigger();
				dep_wait();
				const uint64_t tid = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				const uint64_t pairs = n >> 1;
				const unsigned int it = *iter_counter;
				const bool first = it == 0u;
				if( hist_rr != nullptr && tid == 0 && it > 0u ) {
					hist_rr[ it - 1u ] = scalars[ S_RR ];
					hist_pq[ it - 1u ] = scalars[ S_PQ ];
				}
				// cg.hpp:118  waxpby( p, 1.0, z, 0.0, z )  /  cg.hpp:120  waxpby( p, 1.0, z, rho / rho_prev, p )
				const double beta = first ? 0.0 : __ddiv_rn( scalars[ S_RHO ], scalars[ S_RHO_PREV ] );
				for( uint64_t i = tid; i < pairs; i += stride ) {
					const double2 zv = reinterpret_cast< const double2 * >( z )[ i ];
					const double2 pv = first ? zv : reinterpret_cast< const double2 * >( p )[ i ];
					double2 out;
					out.x = __dadd_rn( __dmul_rn( 1.0, zv.x ), __dmul_rn( beta, pv.x ) );
					out.y = __dadd_rn( __dmul_rn( 1.0, zv.y ), __dmul_rn( beta, pv.y ) );
					reinterpret_cast< double2 * >( p )[ i ] = out;
				}
				if( tid == 0 && ( n & 1 ) ) {
					const double zi = z[ n - 1 ];
					p[ n - 1 ] = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( beta, first ? zi : p[ n - 1 ] ) );
				}
			}

			__global__ void k_cg_update_xr( double * x, double * r, const double * p,
				const double * q, double * scalars, uint64_t n, unsigned int * bump ) {
				dep_trigger();
				dep_wait();
				const uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const double rho = scalars[ S_RHO ];
				const double alpha = __ddiv_rn( rho, scalars[ S_PQ ] ); // cg.hpp:127
				if( i < n ) {
					if( x != nullptr ) { // else: cg.hpp:128 is taken later by k_cg_update_x (cg.cu, lazy x)
						x[ i ] = __dadd_rn( __dmul_rn( 1.0, x[ i ] ), __dmul_rn( alpha, p[ i ] ) );  // cg.hpp:128
					}
					r[ i ] = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -alpha, q[ i ] ) ); // cg.hpp:129
				}
				if( i == 0 ) {
					scalars[ S_RHO_PREV ] = rho; // cg.hpp:130 (nobody reads rho_prev in this launch)
					scalars[ S_ALPHA ] = alpha;
					if( bump != nullptr ) {
						*bump += 1u; // the iteration counter (nobody reads it in this launch)
					}
				}
			}

			// the same update with r'r (cg.hpp:132) reduced in the tree-dot shape on the way out
			// WITH_X false: cg.hpp:128 is taken later by k_cg_update_x (cg.cu, lazy x)
			template< bool WITH_X >
			__global__ void __launch_bounds__( kBlock ) k_cg_update_xr_dot( double * x, double * r, const double * p,
				const double * q, double * scalars, uint64_t n, double * partials, unsigned int * counter, unsigned int * bump ) {
				__shared__ double smem[ 32 ];
				__shared__ bool is_last;
				dep_trigger();
				dep_wait();
				const double rho = scalars[ S_RHO ];
				const double alpha = __ddiv_rn( rho, scalars[ S_PQ ] );
				double acc = 0.0;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				const uint64_t pairs = n >> 1;
				double acc1 = 0.0;
				for( uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x; i < pairs; i += stride ) {
					if( WITH_X ) {
						const double2 xv = reinterpret_cast< const double2 * >( x )[ i ];
						const double2 pv = reinterpret_cast< const double2 * >( p )[ i ];
						double2 xn;
						xn.x = __dadd_rn( __dmul_rn( 1.0, xv.x ), __dmul_rn( alpha, pv.x ) );
						xn.y = __dadd_rn( __dmul_rn( 1.0, xv.y ), __dmul_rn( alpha, pv.y ) );
						reinterpret_cast< double2 * >( x )[ i ] = xn;
					}
					const double2 rv = reinterpret_cast< const double2 * >( r )[ i ];
					const double2 qv = reinterpret_cast< const double2 * >( q )[ i ];
					double2 rn;
					rn.x = __dadd_rn( __dmul_rn( 1.0, rv.x ), __dmul_rn( -alpha, qv.x ) );
					rn.y = __dadd_rn( __dmul_rn( 1.0, rv.y ), __dmul_rn( -alpha, qv.y ) );
					reinterpret_cast< double2 * >( r )[ i ] = rn;
					acc = __dadd_rn( acc, __dmul_rn( rn.x, rn.x ) );
					acc1 = __dadd_rn( acc1, __dmul_rn( rn.y, rn.y ) );
				}
				if( blockIdx.x == 0 && threadIdx.x == 0 && ( n & 1 ) ) {
					const uint64_t i = n - 1;
					if( WITH_X ) {
						x[ i ] = __dadd_rn( __dmul_rn( 1.0, x[ i ] ), __dmul_rn( alpha, p[ i ] ) );
					}
					const double rn = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -alpha, q[ i ] ) );
					r[ i ] = rn;
					acc1 = __dadd_rn( acc1, __dmul_rn( rn, rn ) );
				}
				acc = __dadd_rn( acc, acc1 );
				if( blockIdx.x == 0 && threadIdx.x == 0 ) {
					scalars[ S_RHO_PREV ] = rho;
					scalars[ S_ALPHA ] = alpha;
					if( bump != nullptr ) {
						*bump += 1u;
					}
				}
				grid_tree_finish( block_tree_sum( acc, smem ), partials, counter, scalars + S_RR, smem, &is_last );
			}

			// cg.hpp:128 of the PREVIOUS iteration (cg.cu, lazy x): x <- x + alpha p with the alpha that iteration's r update
			// left in S_ALPHA. Nothing inside an iteration reads x, and p keeps its value until the next p update, so this
			// pass runs on a side stream under the latency-bound coarse levels of the next V-cycle. A small grid with
			// four 16-byte loads per array in flight per thread: enough for a third of the HBM rate, few enough blocks to
			// leave the SMs to the V-cycle. The first iteration has nothing pending.
			__global__ void __launch_bounds__( kBlock ) k_cg_update_x( double * x, const double * p, const double * scalars,
				const unsigned int * iter_counter, uint64_t n ) {
				dep_trigger();
				dep_wait();
				if( *iter_counter == 0u ) {
					return;
				}
				const double alpha = scalars[ S_ALPHA ];
				const uint64_t tid = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				const uint64_t pairs = n >> 1;
				double2 * const x2 = reinterpret_cast< double2 * >( x );
				const double2 * const p2 = reinterpret_cast< const double2 * >( p );
				uint64_t i = tid;
				for( ; i + 3 * stride < pairs; i += 4 * stride ) {
					double2 xv[ 4 ], pv[ 4 ];
					#pragma unroll
					for( int k = 0; k < 4; ++k ) {
						xv[ k ] = x2[ i + k * stride ];
						pv[ k ] = p2[ i + k * stride ];
					}
					#pragma unroll
					for( int k = 0; k < 4; ++k ) {
						xv[ k ].x = __dadd_rn( __dmul_rn( 1.0, xv[ k ].x ), __dmul_rn( alpha, pv[ k ].x ) );
						xv[ k ].y = __dadd_rn( __dmul_rn( 1.0, xv[ k ].y ), __dmul_rn( alpha, pv[ k ].y ) );
						x2[ i + k * stride ] = xv[ k ];
					}
				}
				for( ; i < pairs; i += stride ) {
					double2 xv = x2[ i ];
					const double2 pv = p2[ i ];
					xv.x = __dadd_rn( __dmul_rn( 1.0, xv.x ), __dmul_rn( alpha, pv.x ) );
					xv.y = __dadd_rn( __dmul_rn( 1.0, xv.y ), __dmul_rn( alpha, pv.y ) );
					x2[ i ] = xv;
				}
				if( tid == 0 && ( n & 1 ) ) {
					x[ n - 1 ] = __dadd_rn( __dmul_rn( 1.0, x[ n - 1 ] ), __dmul_rn( alpha, p[ n - 1 ] ) );
				}
			}

			__global__ void k_cg_record( const double * scalars, double * hist_rr, double * hist_pq,
				unsigned int * iter_counter ) {
				dep_trigger();
				dep_wait();
				const unsigned int it = *iter_counter;
				hist_rr[ it ] = scalars[ S_RR ];
				hist_pq[ it ] = scalars[ S_PQ ];
				*iter_counter = it + 1;
			}

			// the same bookkeeping one step late (cg.cu, solves on a communicator): the r'r an iteration leaves behind is
			// only global after the NEXT iteration's combined allreduce, so iteration k records iteration k-1
			__global__ void k_cg_record_deferred( const double * scalars, double * hist_rr, double * hist_pq, unsigned int * iter_counter, int last ) {
				dep_trigger();
				dep_wait();
				const unsigned int it = *iter_counter;
				if( it > 0u ) {
					hist_rr[ it - 1u ] = scalars[ S_RR ];
					hist_pq[ it - 1u ] = scalars[ S_PQ ];
				}
				if( !last ) {
					*iter_counter = it + 1u;
				}
			}

		} // namespace

		// ================================================================ wrappers

		namespace {
			// grid of the vector kernels that move two elements per thread and iteration: one pass for short
			// vectors, a grid-stride loop of about four iterations per thread for long ones
			unsigned int vector_grid( uint64_t n ) {
				const uint64_t pairs = ( n + 1 ) >> 1;
				const uint64_t want = ( pairs + kBlock * 4 - 1 ) / ( kBlock * 4 );
				const uint64_t floor_blocks = ( pairs + kBlock - 1 ) / kBlock;
				const uint64_t small = floor_blocks < 148 * 4 ? floor_blocks : 148 * 4;
				const uint64_t grid = want > small ? want : small;
				return static_cast< unsigned int >( grid < 1 ? 1 : grid );
			}
		} // namespace

		void fill( cudaStream_t st, double * v, uint64_t n, double value ) {
			if( n == 0 ) {
				return;
			}
			const uint64_t head = ( reinterpret_cast< uintptr_t >( v ) & 15u ) != 0 && n > 0 ? 1 : 0;
			const uint64_t pairs = ( n - head ) >> 1;
			const uint64_t want = ( pairs + kBlock * 4 - 1 ) / ( kBlock * 4 ); // four stores per thread
			const unsigned int grid = static_cast< unsigned int >( want < 1 ? 1 : ( want > 148 * 16 ? 148 * 16 : want ) );
			launch( k_fill, grid, kBlock, st, v, n, value, head );
		}

		void waxpby( cudaStream_t st, double * w, double alpha, const double * x, double beta, const double * y,
			uint64_t n ) {
			if( n == 0 ) {
				return;
			}
			launch( k_waxpby, vector_grid( n ), kBlock, st, w, alpha, x, beta, y, n );
		}

		namespace {
			// products per chunk and stage: as long as three stages of every chunk of the block fit shared memory
			int dot_exact_tile( int cpb ) {
				return cpb <= 12 ? 256 : ( cpb <= 24 ? 128 : 64 );
			}
			size_t dot_exact_smem( int cpb, int tile ) {
				return 128 + ( static_cast< size_t >( kDotStages ) * 2 * cpb * ( tile + 2 ) + static_cast< size_t >( 2 ) * cpb * ( tile + 1 ) ) * sizeof( double );
			}
		} // namespace

		void dot_exact_prepare() { // function attributes; outside any stream capture
			static bool done = false;
			if( !done ) {
				SLAB_CUDA( cudaFuncSetAttribute( k_dot_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast< int >( 216 * 1024 ) ) );
				done = true;
			}
		}

		void dot_exact( cudaStream_t st, const double * x, const double * y, uint64_t n, double * partials,
			unsigned int * counter, double * out ) {
			if( n == 0 ) {
				launch( k_dot_empty, 1, 1, st, out );
				return;
			}
			// as many chunks per block as spread the chunks over the SMs (at most one per lane of the adding warp)
			const uint64_t nchunks = ( n + kDotChunk - 1 ) / kDotChunk;
			static int sms = 0;
			if( sms == 0 ) {
				int device = 0;
				SLAB_CUDA( cudaGetDevice( &device ) );
				SLAB_CUDA( cudaDeviceGetAttribute( &sms, cudaDevAttrMultiProcessorCount, device ) );
			}
			// two blocks per SM (their adding warps sit on different sub-partitions and fill each other's hand-over gaps):
			// measured 65 against 78 us at 192^3 (tools/exact_dot_tiles.py)
			int cpb = static_cast< int >( ( nchunks + 2 * sms - 1 ) / ( 2 * sms ) );
			cpb = cpb < 1 ? 1 : ( cpb > 32 ? 32 : cpb );
			if( g_dot_cpb > 0 ) {
				cpb = g_dot_cpb > 32 ? 32 : g_dot_cpb;
			}
			const unsigned int grid = static_cast< unsigned int >( ( nchunks + cpb - 1 ) / cpb );
			int tile = dot_exact_tile( cpb );
			if( g_dot_tile > 0 && dot_exact_smem( cpb, g_dot_tile ) <= 216 * 1024 && ( g_dot_tile % 2 ) == 0 ) {
				tile = g_dot_tile;
			}
			cudaLaunchConfig_t cfg{};
			cfg.gridDim = dim3( grid, 1, 1 );
			cfg.blockDim = dim3( kDotThreads, 1, 1 );
			cfg.dynamicSmemBytes = dot_exact_smem( cpb, tile );
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
			SLAB_CUDA( cudaLaunchKernelEx( &cfg, k_dot_exact, x, y, n, cpb, tile, partials, counter, out ) );
			count_launch();
		}

		uint64_t dot_tree_blocks( uint64_t n, int sm_count ) {
			const uint64_t want = ( n + kBlock * 4 - 1 ) / ( kBlock * 4 );
			const uint64_t cap = static_cast< uint64_t >( sm_count ) * 8;
			const uint64_t blocks = want < cap ? want : cap;
			return blocks < 1 ? 1 : blocks;
		}

		void dot_tree( cudaStream_t st, const double * x, const double * y, uint64_t n, int sm_count, double * partials,
			unsigned int * counter, double * out ) {
			if( n == 0 ) {
				launch( k_dot_empty, 1, 1, st, out );
				return;
			}
			const unsigned int blocks = static_cast< unsigned int >( dot_tree_blocks( n, sm_count ) );
			launch( k_dot_tree, blocks, kBlock, st, x, y, n, partials, counter, out );
		}

		uint64_t spmv_dot_blocks( int64_t nrows ) {
			return blocks_for( nrows > 0 ? nrows : 1, 128 ); // the smallest block any product kernel runs with
		}

		void sum_partials( cudaStream_t st, const double * partials, uint64_t count, double * out ) {
			launch( k_sum_partials, 1, 1024, st, partials, count, out );
		}

		namespace {
			inline bool run_packed( const Sell & S, int64_t rows ) {
				return S.plain_dropped() || ( g_use_packed && S.packed.usable() && rows >= g_packed_min_rows );
			}
		} // namespace

		void spmv( cudaStream_t st, const Sell & S, const double * x, double * y, int64_t nrows, double * dot_partials,
			unsigned int * dot_counter, double * dot_out ) {
			if( nrows == 0 ) {
				if( dot_out != nullptr ) {
					launch( k_dot_empty, 1, 1, st, dot_out );
				}
				return;
			}
			if( run_packed( S, nrows ) ) {
				spmv_packed( st, S, x, y, nullptr, nrows, dot_partials, dot_out );
				return;
			}
			const int64_t * slice_off = S.slice_off;
			const double * vals = S.vals;
			const int32_t * cols = S.cols;
			if( nrows >= g_stream_rows ) {
				const unsigned int grid = blocks_for( nrows );
				switch( g_stream_variant ) {
					case 1:
						launch( k_spmv_batched< 9, 4 >, grid, kBlock, st, slice_off, vals, cols, x, y, nrows, dot_partials, dot_counter, dot_out );
						break;
					case 2:
						launch( k_spmv_batched< 9, 5 >, grid, kBlock, st, slice_off, vals, cols, x, y, nrows, dot_partials, dot_counter, dot_out );
						break;
					case 3:
						launch( k_spmv_batched< 14, 3 >, grid, kBlock, st, slice_off, vals, cols, x, y, nrows, dot_partials, dot_counter, dot_out );
						break;
					case 4:
						launch( k_spmv_batched< 5, 6 >, grid, kBlock, st, slice_off, vals, cols, x, y, nrows, dot_partials, dot_counter, dot_out );
						break;
					case 5:
						launch( k_spmv_batched< 7, 5 >, grid, kBlock, st, slice_off, vals, cols, x, y, nrows, dot_partials, dot_counter, dot_out );
						break;
					default:
						launch( k_spmv_batched< 9, 5 >, grid, kBlock, st, slice_off, vals, cols, x, y, nrows, dot_partials, dot_counter, dot_out );
				}
				if( dot_out != nullptr ) {
					launch( k_sum_partials, 1, 1024, st, static_cast< const double * >( dot_partials ), static_cast< uint64_t >( grid ), dot_out );
				}
				return;
			}
			launch( k_spmv< false >, blocks_for( nrows ), kBlock, st, slice_off, vals, cols, x, y,
				static_cast< const int32_t * >( nullptr ), nrows, dot_partials, dot_counter, dot_out );
			if( dot_out != nullptr ) {
				launch( k_sum_partials, 1, 1024, st, static_cast< const double * >( dot_partials ),
					static_cast< uint64_t >( blocks_for( nrows ) ), dot_out );
			}
		}

		void spmv_masked( cudaStream_t st, const Sell & S, const double * x, double * y, const int32_t * members,
			int64_t count ) {
			if( count == 0 ) {
				return;
			}
			if( run_packed( S, count ) ) {
				spmv_packed( st, S, x, y, members, count, nullptr, nullptr );
				return;
			}
			const int64_t * slice_off = S.slice_off;
			const double * vals = S.vals;
			const int32_t * cols = S.cols;
			launch( k_spmv< true >, blocks_for( count ), kBlock, st, slice_off, vals, cols, x, y, members, count,
				static_cast< double * >( nullptr ), static_cast< unsigned int * >( nullptr ), static_cast< double * >( nullptr ) );
		}

		bool gs_color_step_can_fuse_residual( const Sell & S, int64_t pos_count ) {
			// the packed and the preload shapes keep the matrix row in registers
			return run_packed( S, pos_count ) || pos_count < g_stream_rows;
		}

		void gs_color_step( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t pos_begin, int64_t pos_count,
			double * z, const double * r, int flags, const double * src, double * out, double * zero, size_t window_bytes,
			const int32_t * pos_list, const uint8_t * skip ) {
			if( pos_count == 0 ) {
				return;
			}
			if( run_packed( S, pos_count ) ) {
				gs_color_step_packed( st, S, rows, pos_begin, pos_count, z, r, flags, src, out, zero, pos_list, skip );
				return;
			}
			const int64_t * slice_off = S.slice_off;
			const double * vals = S.vals;
			const int32_t * cols = S.cols;
			if( pos_count >= g_stream_rows ) {
				if( flags & 6 ) {
					fail( SLAB_ERR_INTERNAL, "gs_color_step: the streaming shape cannot fuse the residual or repeat a step" );
				}
				const double * prolong = ( flags & 1 ) ? src : nullptr;
				const unsigned int grid = blocks_for( pos_count );
				if( g_l2_window && window_bytes > 0 ) {
					t_window_base = z;
					t_window_bytes = window_bytes;
				}
				switch( g_stream_variant ) {
					case 1:
						launch( k_gs_color_batched< 9, 4 >, grid, kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z, r, prolong, pos_list, skip );
						break;
					case 3:
						launch( k_gs_color_batched< 14, 3 >, grid, kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z, r, prolong, pos_list, skip );
						break;
					case 4:
						launch( k_gs_color_batched< 5, 6 >, grid, kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z, r, prolong, pos_list, skip );
						break;
					case 5:
						launch( k_gs_color_batched< 7, 5 >, grid, kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z, r, prolong, pos_list, skip );
						break;
					case 6:
						launch( k_gs_color, grid, kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z, r, flags, src, out, zero, pos_list, skip );
						break;
					default:
						launch( k_gs_color_batched< 9, 5 >, grid, kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z, r, prolong, pos_list, skip );
				}
				return;
			}
			launch( k_gs_color, blocks_for( pos_count ), kBlock, st, slice_off, vals, cols, rows, pos_begin, pos_count, z,
				r, flags, src, out, zero, pos_list, skip );
		}

		void residual_restrict( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t n_coarse, const double * z,
			const double * r, double * r_c, double * zero ) {
			if( n_coarse == 0 ) {
				return;
			}
			if( run_packed( S, n_coarse ) ) {
				residual_restrict_packed( st, S, rows, n_coarse, z, r, r_c, zero );
				return;
			}
			const int64_t * slice_off = S.slice_off;
			const double * vals = S.vals;
			const int32_t * cols = S.cols;
			if( n_coarse >= g_stream_rows ) {
				launch( k_residual_restrict_stream, blocks_for( n_coarse ), kBlock, st, slice_off, vals, cols, rows, n_coarse,
					z, r, r_c, zero );
				return;
			}
			launch( k_residual_restrict, blocks_for( n_coarse ), kBlock, st, slice_off, vals, cols, rows, n_coarse, z, r,
				r_c, zero );
		}

		void prolong_add( cudaStream_t st, const int32_t * rows, int64_t n_coarse, double * z, const double * z_c ) {
			if( n_coarse == 0 ) {
				return;
			}
			launch( k_prolong_add, blocks_for( n_coarse ), kBlock, st, rows, n_coarse, z, z_c );
		}

		void cg_update_p( cudaStream_t st, double * p, const double * z, const double * scalars,
			const unsigned int * iter_counter, uint64_t n, double * hist_rr, double * hist_pq ) {
			launch( k_cg_update_p, n == 0 ? 1u : vector_grid( n ), kBlock, st, p, z, scalars, iter_counter, n, hist_rr, hist_pq );
		}

		void cg_update_xr( cudaStream_t st, double * x, double * r, const double * p, const double * q, double * scalars,
			uint64_t n, unsigned int * bump ) {
			launch( k_cg_update_xr, n == 0 ? 1u : blocks_for( n ), kBlock, st, x, r, p, q, scalars, n, bump );
		}

		void cg_update_x( cudaStream_t st, double * x, const double * p, const double * scalars, const unsigned int * iter_counter,
			uint64_t n, int sm_count ) {
			if( n == 0 ) {
				return;
			}
			const uint64_t pairs = ( n + 1 ) >> 1;
			const uint64_t want = ( pairs + kBlock * 4 - 1 ) / ( kBlock * 4 );
			const uint64_t cap = static_cast< uint64_t >( sm_count > 0 ? sm_count : 148 ) * ( g_lazy_x_blocks > 0 ? g_lazy_x_blocks : 1 );
			launch( k_cg_update_x, static_cast< unsigned int >( want < 1 ? 1 : ( want > cap ? cap : want ) ), kBlock, st, x, p, scalars,
				iter_counter, n );
		}

		void cg_update_xr_dot( cudaStream_t st, double * x, double * r, const double * p, const double * q, double * scalars,
			uint64_t n, int sm_count, double * partials, unsigned int * counter, unsigned int * bump ) {
			if( x == nullptr ) {
				launch( k_cg_update_xr_dot< false >, static_cast< unsigned int >( dot_tree_blocks( n, sm_count ) ), kBlock, st, x, r, p, q,
					scalars, n, partials, counter, bump );
				return;
			}
			launch( k_cg_update_xr_dot< true >, static_cast< unsigned int >( dot_tree_blocks( n, sm_count ) ), kBlock, st, x, r, p, q,
				scalars, n, partials, counter, bump );
		}

		void cg_record( cudaStream_t st, const double * scalars, double * hist_rr, double * hist_pq,
			unsigned int * iter_counter ) {
			launch( k_cg_record, 1, 1, st, scalars, hist_rr, hist_pq, iter_counter );
		}

		void cg_record_deferred( cudaStream_t st, const double * scalars, double * hist_rr, double * hist_pq, unsigned int * iter_counter, bool last ) {
			launch( k_cg_record_deferred, 1, 1, st, scalars, hist_rr, hist_pq, iter_counter, last ? 1 : 0 );
		}

	} // namespace kern
} // namespace slabgpu
