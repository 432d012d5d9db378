// plane_spmv.cu — y = A x for a regular box matrix (mxv, operations.hpp:164-167) with the input vector staged
// through shared memory by the bulk-async copy engine and every staged value read ONCE per thread.
//
// A "regular" matrix (BoxTile::regular, tile.cu: one value per offset of the 3x3x3 neighbourhood, every row storing
// exactly the offsets that stay inside the box — checked row by row against the coded copy when the matrix is
// built) needs no matrix stream at all: a launch moves 8 bytes of x in and 8 bytes of y out per row.
//
// A thread block owns `ty` whole x-lines of the box and marches along z. The planes it needs arrive as slabs of
// ty + 2 lines in a ring in shared memory (one cp.async.bulk per line, completion counted on the slot's "full"
// mbarrier; the compute warps hand a slot back through its "empty" mbarrier). Slabs are zero-padded — two zero
// columns in front of every line, zero lines and planes outside the box — so an absent neighbour adds v * 0 = +-0
// to a partial sum that started from +0.0, which never changes it (plane.cu has the argument in full).
//
// The row sum of operations.hpp:116-125 runs over ascending columns: the nine entries of plane z-1, then the nine
// of plane z, then the nine of plane z+1. A thread owns six neighbouring columns (x0 .. x0+5) of one line and keeps
// THREE rows of each in flight: when slab P is in its registers (3 lines x 5 aligned 16-byte reads, conflict-free
// because consecutive threads are three 16-byte groups apart) it adds P's nine entries as the LAST nine of row
// z = P-1 (which is then complete and leaves for y), as the MIDDLE nine of row z = P, and as the FIRST nine of row
// z = P+1. Every sum still starts from +0.0 and takes its 27 separately rounded products in ascending column
// order, so y is bit-identical to the coded and plain kernels — but a staged value is read from shared memory
// once per thread and plane instead of three times: 2.5 sixteen-byte reads per row against 12 in a kernel that
// gathers row by row, which is what lets the product run at the HBM rate instead of the shared-memory rate.
//
// Tree-dot mode: x'(A x) rides on the epilogue (cg.hpp:122-123): a block folds its rows' products in a fixed tree,
// the per-block partials are folded in block order by k_sum_partials — run-to-run deterministic.
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "bulk_copy.cuh"
#include "common.hpp"
#include "device_util.cuh"

namespace slabgpu {

	int g_use_spmv_planes = 1;
	int64_t g_spmv_plane_min_rows = 4096; // smaller products stay with the per-row kernels (one wave of tiny blocks)
	int g_spmv_plane_ty = 0, g_spmv_plane_cz = 0, g_spmv_plane_ns = 0;

	namespace kern {

		namespace {

			using namespace dev;

			constexpr int kCols = 6;           // columns per thread: three aligned pairs
			constexpr int kRing = 8;           // most ring slots
			constexpr int kHeader = 512;       // mbarriers and the dot's warp sums in front of the slabs
			constexpr int kMaxComputeT = 512;  // compute threads; one more warp owns the copy engine
			constexpr size_t kSmemMax = 227u * 1024u;

			struct SpmvGeom {
				double v[ 27 ]; // value of each offset, slot = 9 (dz+1) + 3 (dy+1) + (dx+1)
				int lx, ly, lz;
				int nseg;       // six-column segments per line
				int ncompute;   // compute threads (a multiple of 32)
				int pitch;      // doubles per slab line: lx + 2
				int ty, nyt;    // owned lines per block, y tiles
				int cz, nch;    // planes per block, z chunks
				int ns;         // ring slots
			};

			__host__ __device__ inline int slab_elems( const SpmvGeom & G ) {
				return ( G.ty + 2 ) * G.pitch;
			}

			// three entries (one line of one plane) for the six rows of a thread: acc[c] += v[BASE + dx] * e[c + 1 + dx]
			// in ascending dx. UNIT: every off-diagonal value is -1.0, so the product is -e exactly.
			template< bool UNIT, int BASE >
			__device__ __forceinline__ void add_line( double ( &acc )[ kCols ], const double ( &e )[ kCols + 4 ], const SpmvGeom & G ) {
				#pragma unroll
				for( int dx = 0; dx < 3; ++dx ) {
					#pragma unroll
					for( int c = 0; c < kCols; ++c ) {
						const double x = e[ c + 1 + dx ];
						if( UNIT && BASE + dx != 13 ) {
							acc[ c ] = __dadd_rn( acc[ c ], -x );
						} else {
							acc[ c ] = __dadd_rn( acc[ c ], __dmul_rn( G.v[ BASE + dx ], x ) );
						}
					}
				}
			}

			// line L of the slab in registers: the last three-of-nine of row z = P - 1 on that line, the middle ones of
			// row z = P, the first ones of row z = P + 1
			template< bool UNIT, bool DOT, int L >
			__device__ __forceinline__ void slab_line( const double * base, int P, const SpmvGeom & G, bool last, bool mid, bool first, double ( &a0 )[ kCols ],
				double ( &a1 )[ kCols ], double ( &a2 )[ kCols ], double ( &own )[ kCols ] ) {
				double e[ kCols + 4 ];
				const double2 * const q = reinterpret_cast< const double2 * >( base + L * P );
				#pragma unroll
				for( int m = 0; m < ( kCols + 4 ) / 2; ++m ) {
					const double2 w = q[ m ];
					e[ 2 * m ] = w.x;
					e[ 2 * m + 1 ] = w.y;
				}
				if( last ) {
					add_line< UNIT, 18 + 3 * L >( a0, e, G );
				}
				if( mid ) {
					add_line< UNIT, 9 + 3 * L >( a1, e, G );
				}
				if( first ) {
					add_line< UNIT, 3 * L >( a2, e, G );
				}
				if( DOT && L == 1 ) {
					#pragma unroll
					for( int c = 0; c < kCols; ++c ) {
						own[ c ] = e[ c + 2 ];
					}
				}
			}

			template< bool UNIT, bool DOT >
			__global__ void __launch_bounds__( kMaxComputeT + 32, 1 ) k_spmv_planes( const __grid_constant__ SpmvGeom G, const double * x, double * y,
				double * dot_partials ) {
				extern __shared__ __align__( 128 ) unsigned char smem_raw[];
				uint64_t * const full = reinterpret_cast< uint64_t * >( smem_raw );
				uint64_t * const empty = full + kRing;
				double * const slabs = reinterpret_cast< double * >( smem_raw + kHeader );
				double * const red = reinterpret_cast< double * >( smem_raw + 128 ); // 32 doubles
				const int t = threadIdx.x, nt = blockDim.x;
				const int nc = G.ncompute;
				const int P = G.pitch;
				const int se = slab_elems( G );
				const int ns = G.ns;
				const int ytile = blockIdx.x % G.nyt;
				const int chunk = blockIdx.x / G.nyt;
				const int Ya = ytile * G.ty;
				const int zc0 = chunk * G.cz;
				const int czc = min( G.cz, G.lz - zc0 );
				const int nslabs = czc + 2; // planes zc0 - 1 .. zc0 + czc
				const int lx = G.lx, ly = G.ly;
				const size_t plane_elems = static_cast< size_t >( lx ) * ly;

				// the ring starts as zeros; the copies only ever write lines and planes of the box
				{
					double2 * const w = reinterpret_cast< double2 * >( slabs );
					const int count = ( ns * se + 16 ) / 2;
					for( int i = t; i < count; i += nt ) {
						w[ i ] = make_double2( 0.0, 0.0 );
					}
				}
				if( t == 0 ) {
					for( int s = 0; s < ns; ++s ) {
						bulk::mbar_init( full + s, 1u );
						bulk::mbar_init( empty + s, static_cast< unsigned int >( nc / 32 ) );
					}
					bulk::mbar_fence_init();
				}
				bulk::fence_proxy_async();
				__syncthreads();
				dep_trigger();
				dep_wait();

				if( t >= nc ) {
					// ------------------------------------------------ the copy warp
					const int lane = t - nc;
					const int ya = max( Ya - 1, 0 ), yb = min( Ya + G.ty, ly - 1 ); // the lines of a slab that exist
					const unsigned int line_bytes = static_cast< unsigned int >( lx ) * 8u;
					#pragma unroll 1
					for( int g = 0; g < nslabs; ++g ) {
						const int s = g % ns;
						if( g >= ns ) {
							bulk::mbar_wait( empty + s, static_cast< unsigned int >( ( g / ns - 1 ) & 1 ) );
						}
						const int zp = zc0 - 1 + g;
						double * const slab = slabs + static_cast< size_t >( s ) * se;
						if( zp < 0 || zp >= G.lz ) { // a plane outside the box reads as zeros
							if( g >= ns ) {
								double2 * const w = reinterpret_cast< double2 * >( slab );
								for( int i = lane; i < se / 2; i += 32 ) {
									w[ i ] = make_double2( 0.0, 0.0 );
								}
							}
							__syncwarp();
							if( lane == 0 ) {
								bulk::mbar_arrive( full + s );
							}
							continue;
						}
						if( lane == 0 ) {
							bulk::mbar_arrive_expect_tx( full + s, static_cast< unsigned int >( yb - ya + 1 ) * line_bytes );
						}
						__syncwarp();
						double * const dst = slab + static_cast< size_t >( ya - ( Ya - 1 ) ) * P + 2;
						const double * const from = x + ( static_cast< size_t >( zp ) * ly + ya ) * lx;
						for( int l = lane; l <= yb - ya; l += 32 ) {
							bulk::g2s( dst + static_cast< size_t >( l ) * P, from + static_cast< size_t >( l ) * lx, line_bytes, full + s );
						}
					}
					return;
				}

				// ---------------------------------------------------- the compute warps
				const int line = t / G.nseg;          // owned line of the tile
				const int sx = t - line * G.nseg;
				const int x0 = kCols * sx;
				const int yy = Ya + line;
				const bool row_ok = line < G.ty && yy < ly;
				const int off = ( line < G.ty ? line : 0 ) * P + x0; // slab offset of (line yy - 1, column x0 - 2)
				double a0[ kCols ], a1[ kCols ], a2[ kCols ], own[ kCols ], own_next[ kCols ];
				#pragma unroll
				for( int c = 0; c < kCols; ++c ) {
					a0[ c ] = a1[ c ] = a2[ c ] = 0.0;
					own[ c ] = own_next[ c ] = 0.0;
				}
				double dot = 0.0;
				#pragma unroll 1
				for( int g = 0; g < nslabs; ++g ) {
					const int s = g % ns;
					bulk::mbar_wait( full + s, static_cast< unsigned int >( ( g / ns ) & 1 ) );
					const double * const base = slabs + static_cast< size_t >( s ) * se + off;
					const bool last = g >= 2, mid = g >= 1 && g <= czc, first = g < czc;
					slab_line< UNIT, DOT, 0 >( base, P, G, last, mid, first, a0, a1, a2, own_next );
					slab_line< UNIT, DOT, 1 >( base, P, G, last, mid, first, a0, a1, a2, own_next );
					slab_line< UNIT, DOT, 2 >( base, P, G, last, mid, first, a0, a1, a2, own_next );
					__syncwarp();
					if( ( t & 31 ) == 0 ) {
						bulk::mbar_arrive( empty + s ); // the values are in registers: the slot may be refilled
					}
					if( last && row_ok ) { // row z = P - 1 is complete
						const int z = zc0 + g - 2;
						double * const out = y + static_cast< size_t >( z ) * plane_elems + static_cast< size_t >( yy ) * lx + x0;
						#pragma unroll
						for( int m = 0; m < kCols / 2; ++m ) {
							if( x0 + 2 * m < lx ) {
								*reinterpret_cast< double2 * >( out + 2 * m ) = make_double2( a0[ 2 * m ], a0[ 2 * m + 1 ] );
								if( DOT ) {
									dot = __dadd_rn( dot, __dadd_rn( __dmul_rn( own[ 2 * m ], a0[ 2 * m ] ), __dmul_rn( own[ 2 * m + 1 ], a0[ 2 * m + 1 ] ) ) );
								}
							}
						}
					}
					#pragma unroll
					for( int c = 0; c < kCols; ++c ) {
						a0[ c ] = a1[ c ];
						a1[ c ] = a2[ c ];
						a2[ c ] = 0.0;
						if( DOT ) {
							own[ c ] = own_next[ c ]; // this plane's own values: the row they belong to completes with the next slab
						}
					}
				}
				if( DOT ) {
					// the compute warps only (the copy warp has left): a named barrier over nc threads
					#pragma unroll
					for( int o = 16; o > 0; o >>= 1 ) {
						dot = __dadd_rn( dot, __shfl_down_sync( 0xffffffffu, dot, o ) );
					}
					if( ( t & 31 ) == 0 ) {
						red[ t >> 5 ] = dot;
					}
					asm volatile( "bar.sync 1, %0;" ::"r"( nc ) : "memory" );
					if( t < 32 ) {
						double v = t < nc / 32 ? red[ t ] : 0.0;
						#pragma unroll
						for( int o = 16; o > 0; o >>= 1 ) {
							v = __dadd_rn( v, __shfl_down_sync( 0xffffffffu, v, o ) );
						}
						if( t == 0 ) {
							dot_partials[ blockIdx.x ] = v;
						}
					}
				}
			}

			size_t smem_bytes( const SpmvGeom & G ) {
				return static_cast< size_t >( kHeader ) + ( static_cast< size_t >( G.ns ) * slab_elems( G ) + 16 ) * sizeof( double ) + 16;
			}

			bool unit_stencil( const double ( &v )[ 27 ] ) {
				for( int k = 0; k < 27; ++k ) {
					if( k != 13 && v[ k ] != -1.0 ) {
						return false;
					}
				}
				return std::isfinite( v[ 13 ] );
			}

			// tile shape: as many blocks as fill the SMs evenly, lines per block from the thread budget
			bool fill_geom( SpmvGeom & G, const BoxTile & T, int sm_count ) {
				std::memcpy( G.v, T.vals, sizeof( G.v ) );
				G.lx = T.lx;
				G.ly = T.ly;
				G.lz = T.lz;
				G.pitch = T.lx + 2;
				G.nseg = ( T.lx + kCols - 1 ) / kCols;
				if( G.nseg > kMaxComputeT ) {
					return false;
				}
				double best = 0.0;
				bool found = false;
				SpmvGeom pick = G;
				for( int ty : { 1, 2, 3, 4, 6, 8, 12, 16, 24, 32 } ) {
					if( g_spmv_plane_ty > 0 && ty != g_spmv_plane_ty ) {
						continue;
					}
					if( ty > G.ly && ty != 1 && g_spmv_plane_ty == 0 ) {
						continue;
					}
					SpmvGeom C = G;
					C.ty = ty;
					C.nyt = ( G.ly + ty - 1 ) / ty;
					C.ncompute = ( ty * G.nseg + 31 ) / 32 * 32;
					if( C.ncompute > kMaxComputeT ) {
						continue;
					}
					for( int cz : { 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128 } ) {
						if( g_spmv_plane_cz > 0 && cz != g_spmv_plane_cz ) {
							continue;
						}
						if( cz > G.lz && g_spmv_plane_cz == 0 && cz != 2 ) {
							continue;
						}
						C.cz = std::min( cz, G.lz );
						C.nch = ( G.lz + C.cz - 1 ) / C.cz;
						C.ns = g_spmv_plane_ns > 0 ? std::min( g_spmv_plane_ns, kRing ) : 4;
						C.ns = std::max( 2, std::min( C.ns, C.cz + 2 ) );
						const size_t smem = smem_bytes( C );
						if( smem > kSmemMax ) {
							continue;
						}
						// blocks an SM holds at a time: threads (about 110 registers each) and shared memory
						const int threads = C.ncompute + 32;
						int per_sm = static_cast< int >( std::min< size_t >( kSmemMax / smem, static_cast< size_t >( 65536 / ( threads * 112 ) ) ) );
						per_sm = std::max( 1, std::min( per_sm, 8 ) );
						const int64_t blocks = static_cast< int64_t >( C.nyt ) * C.nch;
						const int64_t slots = static_cast< int64_t >( sm_count ) * per_sm;
						const int64_t waves = ( blocks + slots - 1 ) / slots;
						// a wave costs its steps (planes, halo planes, start-up) times the threads an SM steps through (the
						// FP64 pipe is full from about 384 threads on), plus the halo lines it reads
						const double cost = static_cast< double >( waves ) * ( C.cz + 6.0 ) * std::max( per_sm * C.ncompute, 384 ) * ( 1.0 + 0.3 / ty );
						if( !found || cost < best ) {
							best = cost;
							pick = C;
							found = true;
						}
					}
				}
				if( found ) {
					G = pick;
				}
				return found;
			}

			using SpmvKernel = void ( * )( const SpmvGeom, const double *, double *, double * );

			SpmvKernel pick_kernel( bool unit, bool dot ) {
				if( unit ) {
					return dot ? k_spmv_planes< true, true > : k_spmv_planes< true, false >;
				}
				return dot ? k_spmv_planes< false, true > : k_spmv_planes< false, false >;
			}

			void allow_big_smem() {
				static bool done = false;
				if( !done ) {
					for( int u = 0; u < 2; ++u ) {
						for( int d = 0; d < 2; ++d ) {
							SLAB_CUDA( cudaFuncSetAttribute( pick_kernel( u != 0, d != 0 ), cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast< int >( kSmemMax ) ) );
						}
					}
					done = true;
				}
			}

		} // namespace

		bool spmv_planes_usable( const BoxTile & T, int64_t rows, int sm_count ) {
			if( !g_use_spmv_planes || !T.usable() || !T.regular || rows < g_spmv_plane_min_rows || ( T.lx % 2 ) != 0 || T.lx < 4 || T.ly < 4 || T.lz < 4 ) {
				return false;
			}
			SpmvGeom G{};
			return fill_geom( G, T, sm_count );
		}

		void spmv_planes_prepare() {
			allow_big_smem(); // outside any stream capture
		}

		uint64_t spmv_planes_blocks( const BoxTile & T, int sm_count ) {
			SpmvGeom G{};
			if( !fill_geom( G, T, sm_count ) ) {
				return 0;
			}
			return static_cast< uint64_t >( G.nyt ) * G.nch;
		}

		void spmv_planes( cudaStream_t st, int sm_count, const BoxTile & T, const double * x, double * y, double * dot_partials, double * dot_out ) {
			SpmvGeom G{};
			if( !fill_geom( G, T, sm_count ) ) {
				fail( SLAB_ERR_INTERNAL, "spmv_planes: no tile shape fits this matrix" );
			}
			allow_big_smem();
			const unsigned int grid = static_cast< unsigned int >( G.nyt ) * static_cast< unsigned int >( G.nch );
			const unsigned int block = static_cast< unsigned int >( G.ncompute + 32 );
			const bool unit = unit_stencil( G.v );
			if( std::getenv( "SLAB_PLANE_DEBUG" ) ) {
				std::fprintf( stderr, "spmv_planes box %dx%dx%d: ty %d cz %d ns %d nseg %d block %u grid %u smem %zu unit %d\n", G.lx, G.ly, G.lz, G.ty, G.cz,
					G.ns, G.nseg, block, grid, smem_bytes( G ), unit ? 1 : 0 );
			}
			cudaLaunchConfig_t cfg{};
			cfg.gridDim = dim3( grid, 1, 1 );
			cfg.blockDim = dim3( block, 1, 1 );
			cfg.dynamicSmemBytes = smem_bytes( G );
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
			SLAB_CUDA( cudaLaunchKernelEx( &cfg, pick_kernel( unit, dot_out != nullptr ), G, x, y, dot_partials ) );
			count_launch();
			if( dot_out != nullptr ) {
				sum_partials( st, dot_partials, grid, dot_out );
			}
		}

	} // namespace kern

} // namespace slabgpu
