// sweep_cluster.cu — a whole symmetric Gauss-Seidel sweep of a SMALL level in one launch.
//
// Why. A colour step of a coarse level is a few hundred to a few thousand rows: its kernel runs at the floor
// of a dependent launch (2.2 us on B200 inside a CUDA graph with programmatic launches), and a symmetric sweep
// is fifteen of them (smoother.hpp:108-111). Here ONE launch walks the colours of the sweep itself. Everything a
// row needs that the sweep does not change — its codes, its row index, r[i] — sits in shared memory from the
// prologue on (the matrix part is fetched before the wait on the previous kernel), and so does z; a phase is
// barrier -> shared-memory gathers -> the row's add chain and divide -> barrier. Global memory sees z again at
// the end.
//
// Same arithmetic per row, same colour order as the per-colour launches (k_gs_color_packed in packed.cu):
// rows of one colour do not read each other (coloring.hpp:114-158), so the order of rows inside a colour is
// free and the iterates are bit-identical (tests/test_gpu_cluster_sweep.py). The grid transfers ride on the
// first and last step exactly as they do there (flags bit 0 / bit 1).
//
// One CTA (up to 512 rows per colour, one row per thread), __syncthreads between the colours; ON by default for
// levels whose largest colour has at most 384 rows (tuning key "cluster_rows") and that the plane phases of plane.cu
// do not serve (odd or tiny boxes, general matrices): 16^3 4-level solve 10.6 -> 7.0 ms when it was introduced. The
// dictionary is copied to shared memory here, one 16-byte read per entry: the rows of a small level are all boundary
// rows, a warp's codes differ, and constant loads with a different index per lane are replayed per distinct index.
//
// A second mode — one thread-block cluster of up to 16 CTAs, z replicated in every CTA and updated through distributed
// shared memory — was built, measured and REMOVED in round 2: bit-identical but slower than the per-colour launches
// (104^3 20.2 -> 23.1 ms), because `barrier.cluster.arrive.release` (also what cooperative groups' cluster.sync()
// emits) is MEMBAR.ALL.GPU + ERRBAR + CGAERRBAR in front of UCGABAR_ARV and `wait.acquire` adds CCTL.IVALL: a
// device-wide memory barrier per colour, i.e. what a kernel boundary costs. The levels it was meant for now run the
// three-launch plane phases (plane.cu). The template parameter SINGLE below is what is left of it.
#include "kernels.cuh"

#include <algorithm>
#include <type_traits>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"
#include "device_util.cuh"
#include "packed_decode.cuh"

namespace slabgpu {

	// largest colour (rows) of a level that takes the one-launch sweep (one CTA: at most 512); 0 = per-colour
	// launches everywhere
	int64_t g_cluster_rows = 384;

	namespace kern {

		namespace {

			using namespace dev;
			using namespace coded;

			constexpr int kMaxSweepColors = 8;
			constexpr int kMaxClusterCtas = 16;
			constexpr int kSingleBlock = 512;
			constexpr size_t kMaxSweepSmem = 220 * 1024;

			struct SweepColors {
				int32_t pos[ kMaxSweepColors ];   // first position of the colour in the colour-sorted matrix
				int32_t count[ kMaxSweepColors ]; // members
				int32_t ncolors;
				int32_t n;                        // length of z
			};

			// cluster shape for a level: about 64 rows per CTA (a phase is a latency chain, not a throughput problem),
			// power-of-two clusters, one row per thread
			struct SweepShape {
				unsigned int ctas, block;
				size_t smem;
			};
			SweepShape sweep_shape( uint64_t largest, int ncolors, int chunks, uint64_t n ) {
				SweepShape sh{};
				sh.ctas = 1;
				while( largest > static_cast< uint64_t >( kSingleBlock ) && sh.ctas < static_cast< unsigned int >( kMaxClusterCtas ) && static_cast< uint64_t >( sh.ctas ) * 64u < largest ) {
					sh.ctas *= 2;
				}
				const unsigned int per_cta = static_cast< unsigned int >( ( largest + sh.ctas - 1 ) / sh.ctas );
				sh.block = std::max( 32u, ( per_cta + 31u ) / 32u * 32u );
				sh.smem = static_cast< size_t >( ncolors ) * sh.block * ( 16u * chunks + 8u + 4u ) + 8u * ( n + 2 ); // + 2: the swizzle may index one past an odd n
				return sh;
			}

			__device__ __forceinline__ void cluster_arrive() {
				asm volatile( "barrier.cluster.arrive.release;" ::: "memory" );
			}
			__device__ __forceinline__ void cluster_wait() {
				asm volatile( "barrier.cluster.wait.acquire;" ::: "memory" );
			}
			template< bool SINGLE >
			__device__ __forceinline__ void phase_barrier() {
				if( SINGLE ) {
					__syncthreads();
				} else {
					cluster_arrive();
					cluster_wait();
				}
			}
			// store v at the same shared-memory offset of CTA `rank` of the cluster
			__device__ __forceinline__ void remote_store( uint32_t local_addr, unsigned int rank, double v ) {
				uint32_t remote;
				asm volatile( "mapa.shared::cluster.u32 %0, %1, %2;" : "=r"( remote ) : "r"( local_addr ), "r"( rank ) );
				asm volatile( "st.shared::cluster.f64 [%0], %1;" :: "r"( remote ), "d"( v ) : "memory" );
			}

			// z in shared memory is stored swizzled: the rows of a colour are two elements apart, so the 16 lanes of a
			// half-warp would hit only every other 8-byte slot of a 128-byte line (2-way conflicts on top of the two
			// halves); flipping the lowest index bit in every other group of 16 spreads them over all slots.
			__device__ __forceinline__ int swz( int j ) {
				return j ^ ( ( j >> 4 ) & 1 );
			}

			// ordered row sum of a coded row (operations.hpp:116-125; same products, same order as coded_row_sum in
			// packed_decode.cuh) from the shared-memory copies: one 16-byte read per dictionary entry, one swizzled
			// 8-byte read per gathered element. Levels with escaped rows do not come here.
			template< int NCODES, int CHUNKS >
			__device__ __forceinline__ double sweep_row_sum( const RowCodes< CHUNKS > & rc, int32_t i, const double * s_z,
				const uint4 * s_dict ) {
				constexpr int WORDS = ( NCODES + 3 ) / 4;
				double acc = 0.0;
				#pragma unroll
				for( int wi = 0; wi < WORDS; ++wi ) {
					const unsigned int word = rc.word( wi );
					#pragma unroll
					for( int j = 0; j < 4; ++j ) {
						if( 4 * wi + j < NCODES ) {
							const unsigned int code = ( word >> ( 8 * j ) ) & 0xffu;
							const uint4 e = s_dict[ code ];
							const double val = __hiloint2double( static_cast< int >( e.y ), static_cast< int >( e.x ) );
							const double xv = s_z[ swz( i + static_cast< int >( e.z ) ) ];
							const double prod = __dmul_rn( val, xv );
							if( code != 0u ) { // padding adds nothing
								acc = __dadd_rn( acc, prod );
							}
						}
					}
				}
				return acc;
			}

			// Shared memory of a CTA:
			//   [colour][chunk][thread] uint4 | [colour][thread] double | [colour][thread] int32   the part of its rows' work that
			//       the sweep does not change (codes, r[i], row index), filled once in the prologue — the matrix part before
			//       the wait on the previous kernel;
			//   [n] double   a full copy of z. Every CTA gathers from its own copy; a row's new value is stored into every
			//       CTA's copy through distributed shared memory, and the cluster barrier between two colours orders those
			//       stores against the next colour's gathers. Global memory sees z again only at the end.
			extern __shared__ uint4 sweep_smem[];

			// steps of the sweep: colours 0..nc-1, then nc-2..0; the step of colour nc-1 applies its update twice
			// (the last colour of the forward sweep is the first of the backward sweep, smoother.hpp:108-111)
			// SINGLE: the level fits one CTA (at most kSingleBlock rows per colour) — no cluster, no distributed stores, and
			// the barrier between two colours is the CTA's own (BAR.SYNC, tens of cycles)
			template< int NCODES, int CHUNKS, int BATCH, int DICT, bool SINGLE >
			__global__ void __launch_bounds__( SINGLE ? kSingleBlock : kBlock ) k_gs_sweep_cluster( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const int32_t * __restrict__ rows,
				const __grid_constant__ SweepColors sc, double * z, const double * r, int first_flags, int last_flags,
				const double * src, double * out, double * zero ) {
				const int tx = static_cast< int >( threadIdx.x );
				const int B = static_cast< int >( blockDim.x );
				const unsigned int rank = blockIdx.x; // one cluster: the CTA's rank in it
				const unsigned int ctas = gridDim.x;
				const int t = static_cast< int >( rank ) * B + tx;
				const int nc = sc.ncolors;
				const int nsteps = 2 * nc - 1;
				// the dictionary in shared memory: small levels are all boundary, the codes of a warp's rows differ, and
				// constant loads with a different index per lane are replayed once per distinct index
				__shared__ uint4 s_dict[ DICT ]; // {value low, value high, offset, -}
				for( int k = tx; k < DICT; k += B ) {
					const double v = dp.e[ k ].val;
					s_dict[ k ] = make_uint4( static_cast< unsigned int >( __double2loint( v ) ), static_cast< unsigned int >( __double2hiint( v ) ),
						static_cast< unsigned int >( dp.e[ k ].delta ), 0u );
				}
				uint4 * s_codes = sweep_smem;
				double * s_r = reinterpret_cast< double * >( s_codes + nc * CHUNKS * B );
				int32_t * s_i = reinterpret_cast< int32_t * >( s_r + nc * B );
				double * s_z = reinterpret_cast< double * >( s_i + nc * B );
				{
					// all loads of all colours go out together (unrolled: a rolled loop would wait for each colour's data
					// before asking for the next)
					int32_t row_of[ kMaxSweepColors ];
					RowCodes< CHUNKS > rc_of[ kMaxSweepColors ];
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						row_of[ c ] = -1;
						if( c < nc && t < sc.count[ c ] ) {
							const int32_t pos = sc.pos[ c ] + t;
							row_of[ c ] = rows != nullptr ? rows[ pos ] : pos;
							codes_load( codes, static_cast< int64_t >( pos ), rc_of[ c ] );
						}
					}
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						if( c < nc ) {
							s_i[ c * B + tx ] = row_of[ c ];
							if( row_of[ c ] >= 0 ) {
								#pragma unroll
								for( int j = 0; j < CHUNKS; ++j ) {
									s_codes[ ( c * CHUNKS + j ) * B + tx ] = rc_of[ c ].q[ j ];
								}
							}
						}
					}
					dep_trigger();
					dep_wait();
					double r_of[ kMaxSweepColors ];
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						r_of[ c ] = c < nc && row_of[ c ] >= 0 ? r[ row_of[ c ] ] : 0.0;
					}
					for( int j = tx; j < sc.n; j += B ) {
						s_z[ swz( j ) ] = z[ j ];
					}
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						if( c < nc ) {
							s_r[ c * B + tx ] = r_of[ c ];
						}
					}
				}
				// every copy of z complete (and every CTA of the cluster running) before anybody stores into it
				phase_barrier< SINGLE >();
				#pragma unroll 1
				for( int s = 0; s < nsteps; ++s ) {
					const int c = s < nc ? s : nsteps - 1 - s;
					const int32_t i = s_i[ c * B + tx ];
					if( i >= 0 ) {
						RowCodes< CHUNKS > rc;
						#pragma unroll
						for( int j = 0; j < CHUNKS; ++j ) {
							rc.q[ j ] = s_codes[ ( c * CHUNKS + j ) * B + tx ];
						}
						const double ri = s_r[ c * B + tx ];
						const int flags = ( s == 0 ? first_flags : 0 ) | ( s == nsteps - 1 ? last_flags : 0 );
						const int passes = s == nc - 1 ? 2 : 1;
						double zi = s_z[ swz( i ) ];
						if( flags & 1 ) { // multigrid.hpp:76-77 on the injected rows
							const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ t ] ) );
							zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
							s_z[ swz( i ) ] = zi;
						}
						const uint4 de = s_dict[ rc.diag_code() ];
						const double d = __hiloint2double( static_cast< int >( de.y ), static_cast< int >( de.x ) );
						#pragma unroll 1
						for( int pass = 0; pass < passes; ++pass ) { // smoother.hpp:60-72
							const double sum = sweep_row_sum< NCODES, CHUNKS >( rc, i, s_z, s_dict );
							zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -sum ), __dmul_rn( zi, d ) ), d );
							s_z[ swz( i ) ] = zi; // rows of the colour do not read each other: only this thread reads it before the barrier
						}
						if( flags & 2 ) { // multigrid.hpp:100-104 on the injected rows
							const double az = sweep_row_sum< NCODES, CHUNKS >( rc, i, s_z, s_dict );
							const double f = __dadd_rn( __dmul_rn( 1.0, ri ), __dmul_rn( -1.0, az ) );
							out[ t ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
							zero[ t ] = 0.0;
						}
						if( !SINGLE && s + 1 < nsteps ) { // the other copies
							const uint32_t at = static_cast< uint32_t >( __cvta_generic_to_shared( s_z + swz( i ) ) );
							for( unsigned int other = 0; other < ctas; ++other ) {
								if( other != rank ) {
									remote_store( at, other, zi );
								}
							}
						}
					}
					// also after the last step: no CTA may leave while others could still store into its shared memory
					phase_barrier< SINGLE >();
				}
				#pragma unroll 1
				for( int c = 0; c < nc; ++c ) {
					const int32_t i = s_i[ c * B + tx ];
					if( i >= 0 ) {
						z[ i ] = s_z[ swz( i ) ];
					}
				}
			}

			template< int DICT >
			DictParam< DICT > dict_param( const Packed & P ) {
				DictParam< DICT > dp;
				for( int t = 0; t < DICT; ++t ) {
					dp.e[ t ].val = t < P.dict_size ? P.h_dict[ t ].val : 0.0;
					dp.e[ t ].delta = t < P.dict_size ? P.h_dict[ t ].delta : 0;
				}
				return dp;
			}

			template< class... KArgs, class... Args >
			void launch_cluster( void ( *kernel )( KArgs... ), unsigned int ctas, unsigned int block, size_t smem_bytes, cudaStream_t st,
				Args... args ) {
				cudaLaunchConfig_t cfg{};
				cfg.gridDim = dim3( ctas, 1, 1 );
				cfg.blockDim = dim3( block, 1, 1 );
				cfg.dynamicSmemBytes = smem_bytes;
				cfg.stream = st;
				cudaLaunchAttribute attr[ 2 ];
				unsigned int count = 0;
				attr[ count ].id = cudaLaunchAttributeClusterDimension;
				attr[ count ].val.clusterDim.x = ctas;
				attr[ count ].val.clusterDim.y = 1;
				attr[ count ].val.clusterDim.z = 1;
				++count;
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

			template< int N, int D >
			void sweep_launch( cudaStream_t st, const Packed & P, const PlainRef & plain, const int32_t * rows, const SweepColors & sc,
				unsigned int ctas, unsigned int block, size_t smem, double * z, const double * r, int first_flags, int last_flags,
				const double * src, double * out, double * zero ) {
				constexpr int C = ( N + 16 ) / 16;
				if( ctas == 1 ) {
					auto kernel = k_gs_sweep_cluster< N, C, 2, D, true >; // 512 threads: the two-word batches' register count
					static bool prepared = false;
					if( !prepared ) {
						SLAB_CUDA( cudaFuncSetAttribute( kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast< int >( kMaxSweepSmem ) ) );
						prepared = true;
					}
					launch_cluster( kernel, ctas, block, smem, st, P.codes, dict_param< D >( P ), plain, rows, sc, z, r, first_flags,
						last_flags, src, out, zero );
					return;
				}
				// the multi-CTA cluster form (z replicated per CTA, updates through distributed shared memory) was measured
				// and lost to the per-colour launches (file header): it is not instantiated any more
				fail( SLAB_ERR_INTERNAL, "gs_sweep_cluster: the level does not fit one CTA" );
			}

			template< int D >
			void sweep_by_width( cudaStream_t st, const Packed & P, const PlainRef & plain, const int32_t * rows, const SweepColors & sc,
				unsigned int ctas, unsigned int block, size_t smem, double * z, const double * r, int first_flags, int last_flags,
				const double * src, double * out, double * zero ) {
				switch( P.ncodes ) {
					case 8: sweep_launch< 8, D >( st, P, plain, rows, sc, ctas, block, smem, z, r, first_flags, last_flags, src, out, zero ); break;
					case 16: sweep_launch< 16, D >( st, P, plain, rows, sc, ctas, block, smem, z, r, first_flags, last_flags, src, out, zero ); break;
					case 27: sweep_launch< 27, D >( st, P, plain, rows, sc, ctas, block, smem, z, r, first_flags, last_flags, src, out, zero ); break;
					case 32: sweep_launch< 32, D >( st, P, plain, rows, sc, ctas, block, smem, z, r, first_flags, last_flags, src, out, zero ); break;
					case 64: sweep_launch< 64, D >( st, P, plain, rows, sc, ctas, block, smem, z, r, first_flags, last_flags, src, out, zero ); break;
					default: fail( SLAB_ERR_INTERNAL, "packed matrix with an unknown width class" );
				}
			}

		} // namespace

		bool gs_sweep_cluster_usable( const Sell & S, const std::vector< int64_t > & color_pos, const std::vector< uint64_t > & color_size,
			uint64_t n ) {
			if( g_cluster_rows <= 0 || !g_use_packed || !S.packed.usable() || S.packed.escaped_rows != 0 ) {
				return false;
			}
			const size_t nc = color_size.size();
			if( nc < 1 || nc > static_cast< size_t >( kMaxSweepColors ) || color_pos.size() < nc ) {
				return false;
			}
			const uint64_t largest = *std::max_element( color_size.begin(), color_size.end() );
			const int64_t limit = std::min< int64_t >( g_cluster_rows, static_cast< int64_t >( kSingleBlock ) ); // one CTA, one row per thread
			if( largest < 1 || static_cast< int64_t >( largest ) > limit || color_pos[ nc - 1 ] >= ( int64_t( 1 ) << 30 ) ) {
				return false;
			}
			return sweep_shape( largest, static_cast< int >( nc ), S.packed.chunks, n ).smem <= kMaxSweepSmem; // z has to fit
		}

		void gs_sweep_cluster( cudaStream_t st, const Sell & S, const int32_t * rows, const std::vector< int64_t > & color_pos,
			const std::vector< uint64_t > & color_size, uint64_t n, double * z, const double * r, int first_flags, int last_flags,
			const double * src, double * out, double * zero ) {
			const Packed & P = S.packed;
			const PlainRef plain{ S.slice_off, S.vals, S.cols };
			SweepColors sc{};
			sc.ncolors = static_cast< int32_t >( color_size.size() );
			sc.n = static_cast< int32_t >( n );
			uint64_t largest = 1;
			for( int k = 0; k < sc.ncolors; ++k ) {
				sc.pos[ k ] = static_cast< int32_t >( color_pos[ k ] );
				sc.count[ k ] = static_cast< int32_t >( color_size[ k ] );
				largest = std::max( largest, color_size[ k ] );
			}
			const SweepShape sh = sweep_shape( largest, sc.ncolors, P.chunks, n );
			if( P.dict_size <= 32 ) {
				sweep_by_width< 32 >( st, P, plain, rows, sc, sh.ctas, sh.block, sh.smem, z, r, first_flags, last_flags, src, out, zero );
			} else {
				sweep_by_width< 256 >( st, P, plain, rows, sc, sh.ctas, sh.block, sh.smem, z, r, first_flags, last_flags, src, out, zero );
			}
		}

	} // namespace kern
} // namespace slabgpu
